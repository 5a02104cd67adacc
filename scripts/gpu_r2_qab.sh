#!/bin/bash
# A/B of the quantizer: product library vs build/exp_$B, alone and in
# the ResNet-50 step; then the quantizer parity tests on the product library.
cd "${GRAFT_REPO_ROOT:-.}"
B=${B:-noflat}
mkdir -p gpurun_out
for L in prod $B prod $B; do
  if [ $L = prod ]; then LP=""; else LP="AXB_LIB_PATH=build/exp_$L/libaxb.so"; fi
  echo "== $L"; env $LP timeout 300 python scripts/quant_bench.py 2>&1 | tail -18
done
for L in prod $B; do
  if [ $L = prod ]; then LP=""; else LP="AXB_LIB_PATH=build/exp_$L/libaxb.so"; fi
  env $LP timeout 600 python bench.py --steps 5 --no-cpu-baseline --tuned-from build/tuned_r50.json > gpurun_out/bench_qab_$L.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_qab_$L.log').read().strip().splitlines()[-1]); print('$L', d['value'], d['parity']['status'], d['hbm']['kernels']['quantize'])"
done
timeout 900 python -m pytest tests -q -m gpu -x -k "quant or graph or golden or r50 or cx_output or r8" > gpurun_out/pytest_qab.txt 2>&1; tail -2 gpurun_out/pytest_qab.txt
