#!/bin/bash
# ncu --set full captures of the ftable conv kernel: R8 s0b0.a/b, R50 (b64) s0b1.b, s2b1.b, s2b1.c
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
# replay the timed runs' autotuned kernel choices under ncu (its serialised replays distort tuning)
R8T=""; [ -f gpurun_out/tuned_r8.json ] && R8T="--tuned-from gpurun_out/tuned_r8.json"
R50T=""; [ -f gpurun_out/tuned_r50.json ] && R50T="--tuned-from gpurun_out/tuned_r50.json"
TAG=${TAG:-fp}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv_ft -s 1 -c 2 \
    -o gpurun_out/prof_r8_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline $R8T > gpurun_out/ncu_r8_$TAG.log 2>&1
for L in ${R50_LAUNCHES:-6 29}; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s $L -c 1 \
    -o gpurun_out/prof_r50_l${L}_$TAG -f python bench.py --workload r50 --batch 64 --steps 1 --warmup 1 --no-cpu-baseline --no-autotune > gpurun_out/ncu_r50_l${L}_$TAG.log 2>&1
done
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi; true
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lutconv -c 10 \
    --csv --log-file gpurun_out/traffic_r8.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline $R8T > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lutconv -c 54 \
    --csv --log-file gpurun_out/traffic_r50.csv python bench.py --workload r50 --steps 1 --warmup 3 --no-cpu-baseline $R50T > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r8_$TAG.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline $R8T > /dev/null 2>&1
