#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python scripts/variant_matrix.py --workload r50 --nodes stem,s0b0.a,s0b1.b,s0b1.c,s1b1.b,s2b1.a,s2b1.b,s3b0.b,s3b1.b,fc > gpurun_out/matrix_r50_c.jsonl 2>&1
for V in c64_j8_w12_k2 ft16_tm3_w12_k8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 54 -c 1 -o gpurun_out/prof_r50_s0b1b_$V -f \
      python scripts/ft_one.py --workload r50 --batch 64 --node s0b1.b --variant $V --reps 1 > gpurun_out/ncu_$V.log 2>&1
done
