#!/bin/bash
# Round-2 evidence in one gpurun call (outputs under gpurun_out/, collected into profiles/ by
# scripts/collect_r2.sh TAG):
#   GPU tests + smoke; bench lines: ResNet-50 b256 (default, with the CPU baseline), ResNet-8, MobileNet,
#   ResNet-62 sweep, the reference arm; per-layer tables + autotuned picks + RunReports;
#   ncu --set full digests of the CX conv on ResNet-50 (3x3 s0b1.b, 1x1 s1b1.c) and ResNet-8 (s0b0.b);
#   the launch list of one ResNet-50 step and DRAM traffic per conv launch (replaying the tuned picks).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$T.txt
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1; tail -1 gpurun_out/smoke_$T.txt
timeout 900 python bench.py --steps 10 --layers-out gpurun_out/layers_r50_$T.json --tuned-out gpurun_out/tuned_r50_$T.json \
    --report-out gpurun_out/report_r50_$T > gpurun_out/bench_r50_$T.log 2>&1; tail -1 gpurun_out/bench_r50_$T.log > gpurun_out/bench_r50_$T.json
timeout 600 python bench.py --workload r8 --steps 20 --no-cpu-baseline --layers-out gpurun_out/layers_r8_$T.json \
    --tuned-out gpurun_out/tuned_r8_$T.json --report-out gpurun_out/report_r8_$T > gpurun_out/bench_r8_$T.log 2>&1
tail -1 gpurun_out/bench_r8_$T.log > gpurun_out/bench_r8_$T.json
timeout 600 python bench.py --workload mbv1 --steps 10 --no-cpu-baseline --layers-out gpurun_out/layers_mbv1_$T.json \
    > gpurun_out/bench_mbv1_$T.log 2>&1; tail -1 gpurun_out/bench_mbv1_$T.log > gpurun_out/bench_mbv1_$T.json
timeout 900 python bench.py --workload r62sweep --steps 2 --no-cpu-baseline > gpurun_out/bench_r62sweep_$T.log 2>&1
tail -1 gpurun_out/bench_r62sweep_$T.log > gpurun_out/bench_r62sweep_$T.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$T.log 2>&1
tail -1 gpurun_out/bench_ref_$T.log > gpurun_out/bench_ref_$T.json
TUNED=gpurun_out/tuned_r50_$T.json
for NV in s0b1.b s1b1.c; do
  V=$(python -c "import json; print(json.load(open('$TUNED'))['$NV'])")
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 54 -c 1 -o gpurun_out/prof_${T}_$NV -f \
      python scripts/ft_one.py --workload r50 --node $NV --variant $V --reps 1 > gpurun_out/ncu_${T}_$NV.log 2>&1
  python scripts/ncu_summary.py --rep gpurun_out/prof_${T}_$NV.ncu-rep --out gpurun_out/ncusum_${T}_$NV.md > /dev/null 2>&1
  python scripts/ncu_digest.py gpurun_out/prof_${T}_$NV.ncu-rep --out gpurun_out/ncudig_${T}_$NV.md > /dev/null 2>&1
done
V=$(python -c "import json; print(json.load(open('gpurun_out/tuned_r8_$T.json'))['s0b0.b'])")
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 10 -c 1 -o gpurun_out/prof_${T}_r8s0b0b -f \
    python scripts/ft_one.py --workload r8 --node s0b0.b --variant $V --reps 1 > gpurun_out/ncu_${T}_r8.log 2>&1
python scripts/ncu_summary.py --rep gpurun_out/prof_${T}_r8s0b0b.ncu-rep --out gpurun_out/ncusum_${T}_r8s0b0b.md > /dev/null 2>&1
python scripts/ncu_digest.py gpurun_out/prof_${T}_r8s0b0b.ncu-rep --out gpurun_out/ncudig_${T}_r8s0b0b.md > /dev/null 2>&1
rm -f gpurun_out/prof_${T}_r8s0b0b.ncu-rep gpurun_out/prof_${T}_s1b1.c.ncu-rep
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50_$T.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --tuned-from $TUNED > /dev/null 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lutconv -c 54 \
    --csv --log-file gpurun_out/traffic_r50_$T.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
    --tuned-from $TUNED > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:lutconv -c 10 \
    --csv --log-file gpurun_out/traffic_r8_$T.csv python bench.py --workload r8 --steps 1 --warmup 3 --no-cpu-baseline \
    --tuned-from gpurun_out/tuned_r8_$T.json > /dev/null 2>&1
du -sh gpurun_out
# one-rank torchrun launch: NCCL communicator + the logits/counts exchange on the device (INIT log kept)
timeout 900 python bench.py --gpus 1 --launch --steps 5 --no-cpu-baseline --tuned-from $TUNED \
    > gpurun_out/bench_r50_nccl_$T.log 2> gpurun_out/nccl_init_$T.log
tail -1 gpurun_out/bench_r50_nccl_$T.log > gpurun_out/bench_r50_nccl_$T.json
# nondeterminism stress of every ftable-kernel variant (compute-sanitizer is closed on this pool)
timeout 900 python scripts/ft_stress.py 10 > gpurun_out/ft_stress_$T.txt 2>&1
tail -3 gpurun_out/ft_stress_$T.txt
