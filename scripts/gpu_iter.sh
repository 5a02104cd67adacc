#!/bin/bash
# test + tune + bench + ncu of one main layer
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-it}
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_$TAG.txt
if [ -n "$TUNE" ]; then
  timeout 900 python scripts/tune_variants.py --workload r8 $TUNE --out gpurun_out/tune_r8_$TAG.json > /dev/null 2>&1
  timeout 900 python scripts/tune_variants.py --workload r50 --batch 128 $TUNE --out gpurun_out/tune_r50_$TAG.json > /dev/null 2>&1
fi
timeout 600 python bench.py --steps 20 --warmup 3 --layers-out gpurun_out/layers_r8_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r8_$TAG.txt
timeout 900 python bench.py --workload r50 --steps 3 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r50_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r8_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lutconv_fast -s ${NCU_SKIP:-1} -c ${NCU_COUNT:-2} \
    -o gpurun_out/prof_r8_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r8_$TAG.log 2>&1
fi
