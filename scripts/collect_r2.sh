#!/bin/bash
# Copy one gpu_r2_round.sh run (TAG) from gpurun_out/ into profiles/ as r2_<TAG>_*: bench lines, per-layer
# tables, tuned picks, run reports, ncu summaries + digests (with the ResNet-50 one-step launch breakdown),
# DRAM traffic per conv launch (profiles/traffic_r50.json).
#   bash scripts/collect_r2.sh r2a
set -e
T=${1:?tag}
cd "$(dirname "$0")/.."
G=gpurun_out
P=profiles
for w in r50 r8 mbv1 r62sweep ref; do cp $G/bench_${w}_$T.json $P/r2_${T}_bench_$w.json; done
for w in r50 r8 mbv1; do cp $G/layers_${w}_$T.json $P/r2_${T}_layers_$w.json; done
for w in r50 r8; do
    cp $G/tuned_${w}_$T.json $P/r2_tuned_$w.json
    cp $G/report_${w}_$T.json $P/r2_${T}_report_$w.json
    cp $G/report_${w}_$T.csv $P/r2_${T}_report_$w.csv
done
cp $G/pytest_gpu_$T.txt $P/r2_${T}_pytest_gpu.txt
cp $G/smoke_$T.txt $P/r2_${T}_smoke.txt
cp $G/launches_r50_$T.csv $P/r2_${T}_launches_r50.csv
for n in s0b1.b s1b1.c r8s0b0b; do
    cat $G/ncusum_${T}_$n.md $G/ncudig_${T}_$n.md > $P/r2_${T}_ncu_$n.md
done
python scripts/step_breakdown.py $G/launches_r50_$T.csv $P/r2_${T}_ncu_s0b1.b.md 108 > /dev/null
python scripts/traffic.py $G/traffic_r50_$T.csv r50
[ -f $G/traffic_r8_$T.csv ] && python scripts/traffic.py $G/traffic_r8_$T.csv r8
[ -f $G/bench_r50_nccl_$T.json ] && cp $G/bench_r50_nccl_$T.json $P/r2_${T}_bench_r50_nccl.json
[ -f $G/nccl_init_$T.log ] && grep -E "NCCL INFO|launching" $G/nccl_init_$T.log | head -60 > $P/r2_${T}_nccl_init.txt
[ -f $G/ft_stress_$T.txt ] && cp $G/ft_stress_$T.txt $P/r2_${T}_ft_stress.txt
echo "collected $T"
