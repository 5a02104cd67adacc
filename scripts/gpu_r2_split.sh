#!/bin/bash
# c64 tail split: parity tests that exercise every ftable variant, then A/B timing split on/off
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "code_major or ftable_variants or autotune or benchmarked" > gpurun_out/pytest_split.txt 2>&1; tail -5 gpurun_out/pytest_split.txt
for NV in ${LAYERS:-s3b1.b:c64_j16_w8_k2 s3b1.b:c64_j8_w12_k2 s2b1.b:c64_j16_w8_k2 s1b1.b:c64_j16_w8_k2 s0b1.b:c64_j16_w8_k2 s2b1.a:c64_j16_w8_k2 s1b1.c:c64_j8_w12_k2 s3b1.a:c64_j16_w8_k2}; do
  N=${NV%%:*}; V=${NV##*:}
  echo "$N $V split: $(timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1)  nosplit: $(AXB_C64_SPLIT=0 timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1)"
done
