#!/bin/bash
# ftable kernel: parity tests, bench r8/r50 (ftable on and off), ncu capture of one ftable launch
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-ft}
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_K:-} 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r8_$TAG.json 2>&1 | tail -2 | tee gpurun_out/bench_r8_$TAG.txt
timeout 900 python bench.py --workload r50 --steps 3 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$TAG.json 2>&1 | tail -2 | tee gpurun_out/bench_r50_$TAG.txt
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv_ft -s ${NCU_SKIP:-1} -c ${NCU_COUNT:-2} \
    -o gpurun_out/prof_r8_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r8_$TAG.log 2>&1
fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi; true
