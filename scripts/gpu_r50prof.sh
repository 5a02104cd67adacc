#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-p}
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 3 --layers-out gpurun_out/layers_r8_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r8_$TAG.txt
timeout 900 python bench.py --workload r50 --steps 3 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r50_$TAG.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r8_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50_$TAG.csv python bench.py --workload r50 --batch 64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lutconv_fast -s 6 -c 1 \
    -o gpurun_out/prof_r50_s0b1b_$TAG -f python bench.py --workload r50 --batch 128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_r50a_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lutconv_fast -s 34 -c 1 \
    -o gpurun_out/prof_r50_s2b1b_$TAG -f python bench.py --workload r50 --batch 128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_r50b_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lutconv_fast -s 1 -c 2 \
    -o gpurun_out/prof_r8_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r8_$TAG.log 2>&1
