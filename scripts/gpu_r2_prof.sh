#!/bin/bash
# Round-2 profiles: ncu --set full of the c64 conv on ResNet-50 layers (digest + summary on the box; one
# .ncu-rep kept), the launch list of one ResNet-50 step, DRAM traffic per conv launch.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
T=${TAG:-p}
for NV in ${LAYERS:-s0b1.b:c64_j16_w8_k2 s1b1.c:c64_j16_w8_k2}; do
  N=${NV%%:*}; V=${NV##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 54 -c 1 -o gpurun_out/prof_${T}_$N -f \
      python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 1 > gpurun_out/ncu_${T}_$N.log 2>&1
  python scripts/ncu_summary.py --rep gpurun_out/prof_${T}_$N.ncu-rep --out gpurun_out/ncusum_${T}_$N.md > /dev/null 2>&1
  python scripts/ncu_digest.py gpurun_out/prof_${T}_$N.ncu-rep --out gpurun_out/ncudig_${T}_$N.md > /dev/null 2>&1
done
if [ -n "$STEP" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50_$T.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tuned-from ${TUNED:-profiles/r2_tuned_r50.json} > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lutconv -c 54 \
    --csv --log-file gpurun_out/traffic_r50_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    --tuned-from ${TUNED:-profiles/r2_tuned_r50.json} > /dev/null 2>&1
fi
du -sh gpurun_out
