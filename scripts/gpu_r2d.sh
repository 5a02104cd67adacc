#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ftable_variants or code_major" > gpurun_out/pytest_d.txt 2>&1; tail -3 gpurun_out/pytest_d.txt
timeout 900 python scripts/variant_matrix.py --workload r50 --nodes stem,s0b0.a,s0b1.b,s0b1.c,s1b1.b,s2b1.a,s2b1.b,s3b1.b --variants c64_j8_w12_k2,c64_j16_w8_k2,c64_j16_w8_k2_c4,c64_j16_w10_k2_c4,c64_j16_w8_k1_c4,ft16_tm3_w12_k8,cm32_j4_w16_k4 > gpurun_out/matrix_r50_d.jsonl 2>&1
tail -3 gpurun_out/matrix_r50_d.jsonl | cut -c1-300
