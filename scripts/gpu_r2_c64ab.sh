#!/bin/bash
# c64 kernel: time with and without the table-stage refills (A/B experiment library), and ncu raw pages
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for NV in s0b1.b:c64_j16_w8_k2 s1b1.c:c64_j8_w12_k2 s0b1.c:c64_j8_w12_k2 s2b1.a:c64_j16_w8_k2 s1b1.b:c64_j16_w8_k2; do
  N=${NV%%:*}; V=${NV##*:}
  echo "$N $V product: $(timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1)"
  echo "$N $V norefill: $(AXB_LIB_PATH=build/exp_norefill/libaxb.so timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1)"
done
for NV in s0b1.b:c64_j16_w8_k2 s1b1.c:c64_j8_w12_k2; do
  N=${NV%%:*}; V=${NV##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lutconv -s 54 -c 1 -o /tmp/prof_$N -f \
      python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 1 > gpurun_out/ncu_${N}.log 2>&1
  ncu -i /tmp/prof_$N.ncu-rep --page raw --csv > gpurun_out/ncuraw_${N}_$V.csv 2>/dev/null
  ncu -i /tmp/prof_$N.ncu-rep --page source --csv --print-source sass > gpurun_out/ncusrc_${N}_$V.csv 2>/dev/null
  python scripts/ncu_summary.py --rep /tmp/prof_$N.ncu-rep --out gpurun_out/ncu_${N}_$V.md > /dev/null 2>&1
done
ls -la gpurun_out | tail -8
