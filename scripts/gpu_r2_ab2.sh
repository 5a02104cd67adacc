#!/bin/bash
# A/B: product library vs an experiment build (build/exp_$B/libaxb.so) on the ResNet-50 step with fixed
# tuned picks (build/tuned_r50.json), alternating, then the GPU tests on the product library.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
B=${B:-nopf}; T=${TAG:-ab}
for r in 1 2; do
  for L in prod $B; do
    if [ $L = prod ]; then LP=""; else LP="AXB_LIB_PATH=build/exp_$L/libaxb.so"; fi
    env $LP timeout 600 python bench.py --steps 5 --no-cpu-baseline --tuned-from build/tuned_r50.json \
      --layers-out gpurun_out/layers_r50_${T}_${L}_$r.json > gpurun_out/bench_r50_${T}_${L}_$r.log 2>&1
    python -c "import json,sys; d=json.loads(open('gpurun_out/bench_r50_${T}_${L}_$r.log').read().strip().splitlines()[-1]); print('$L', $r, d['value'], d['parity']['status'], d['roofline']['frac'])"
  done
done
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$T.txt
