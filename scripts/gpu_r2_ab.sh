#!/bin/bash
# A/B: product library vs experiment libraries (EXPS="tag1 tag2") on R50 layers (LAYERS="node:variant ...")
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for NV in ${LAYERS:-s0b1.b:c64_j16_w8_k2 s1b1.c:c64_j8_w12_k2 s0b1.c:c64_j8_w12_k2 s2b1.a:c64_j16_w8_k2 s1b1.b:c64_j16_w8_k2}; do
  N=${NV%%:*}; V=${NV##*:}
  echo "$N $V product: $(timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1)"
  for E in $EXPS; do
    echo "$N $V $E: $(AXB_LIB_PATH=build/exp_$E/libaxb.so timeout 300 python scripts/ft_one.py --workload r50 --node $N --variant $V --reps 3 2>&1 | tail -1)"
  done
done
