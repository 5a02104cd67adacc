#!/bin/bash
# ncu captures of the LUT conv kernel + launch lists (one GPU, serialised replays).
#   TAG=x bash scripts/gpu_prof.sh
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-p}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r8_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50_$TAG.csv python bench.py --workload r50 --batch 64 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
# R8: launches 1,2 of the first profiled step (s0b0.a, s0b0.b); R50 b128: launch 6 (s0b1.b), 16 (s1b0.b)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lutconv_fast -s ${R8_SKIP:-1} -c 2 \
    -o gpurun_out/prof_r8_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_r8_$TAG.log 2>&1
for L in ${R50_LAUNCHES:-6 16}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lutconv_fast -s $L -c 1 \
    -o gpurun_out/prof_r50_l${L}_$TAG -f python bench.py --workload r50 --batch 128 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_r50_l${L}_$TAG.log 2>&1
done
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi; true
