#!/bin/bash
# Round-2 call b: full GPU tests, R50 per-layer table + picks, ncu of the c64 and pair-major kernels on R50 s0b1.b
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_b.txt 2>&1; tail -5 gpurun_out/pytest_gpu_b.txt
timeout 900 python bench.py --steps 5 --no-cpu-baseline --layers-out gpurun_out/layers_r50_b.json --tuned-out gpurun_out/tuned_r50_b.json > gpurun_out/bench_r50_b.log 2>&1; tail -1 gpurun_out/bench_r50_b.log > gpurun_out/bench_r50_b.json
for V in c64_j8_w16_k2 ft16_tm2_w16_k8 cm32_j4_w16_k4; do
  timeout 300 python scripts/ft_one.py --workload r50 --batch 64 --node s0b1.b --variant $V --reps 3 2>&1 | tail -3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 1 -c 1 -o gpurun_out/prof_r50_s0b1b_$V -f \
      python scripts/ft_one.py --workload r50 --batch 64 --node s0b1.b --variant $V --reps 2 > gpurun_out/ncu_$V.log 2>&1
done
for N in s2b1.b s1b1.c s3b0.b; do
  timeout 300 python scripts/ft_one.py --workload r50 --batch 64 --node $N --variant c64_j8_w16_k2 --reps 3 2>&1 | tail -1
  timeout 300 python scripts/ft_one.py --workload r50 --batch 64 --node $N --variant ft16_tm2_w16_k8 --reps 3 2>&1 | tail -1
done
