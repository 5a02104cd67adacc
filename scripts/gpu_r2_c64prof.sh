#!/bin/bash
# LDS.128 quarter-warp microbenchmark + ncu --set full of the c64 / code-major kernels on ResNet-50 layers
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
./build/lds128_quarters | tee gpurun_out/lds128_quarters.json
timeout 600 python scripts/zp_stats.py --workload r50 --images 2 --out gpurun_out/zp_r50.json > gpurun_out/zp_r50.log 2>&1; tail -1 gpurun_out/zp_r50.log
for NV in s0b1.b:c64_j16_w8_k2 s1b1.c:c64_j8_w12_k2 s0b1.c:cm32_j4_w16_k4 s0b1.c:c64_j8_w12_k2 s2b1.a:c64_j16_w8_k2; do
  N=${NV%%:*}; V=${NV##*:}
  timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 54 -c 1 -o gpurun_out/prof_r50_${N}_$V -f \
      python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 1 > gpurun_out/ncu_${N}_$V.log 2>&1
done
