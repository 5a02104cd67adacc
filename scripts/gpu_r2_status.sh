#!/bin/bash
# Round-2 status call: GPU parity tests, smoke, default bench (ResNet-50 b256) + ResNet-8 + MobileNet lines
# with per-layer tables and autotune picks.  TAG names the outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$T.txt
if [ -z "$NOTEST" ]; then
timeout ${TEST_TIMEOUT:-1500} python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -8 gpurun_out/pytest_gpu_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1; tail -2 gpurun_out/smoke_$T.txt
fi
timeout 900 python bench.py --steps 5 --layers-out gpurun_out/layers_r50_$T.json --tuned-out gpurun_out/tuned_r50_$T.json \
    > gpurun_out/bench_r50_$T.log 2>&1; tail -1 gpurun_out/bench_r50_$T.log > gpurun_out/bench_r50_$T.json
timeout 600 python bench.py --workload r8 --steps 20 --no-cpu-baseline --layers-out gpurun_out/layers_r8_$T.json \
    --tuned-out gpurun_out/tuned_r8_$T.json > gpurun_out/bench_r8_$T.log 2>&1; tail -1 gpurun_out/bench_r8_$T.log > gpurun_out/bench_r8_$T.json
timeout 600 python bench.py --workload mbv1 --steps 5 --no-cpu-baseline --layers-out gpurun_out/layers_mbv1_$T.json \
    > gpurun_out/bench_mbv1_$T.log 2>&1; tail -1 gpurun_out/bench_mbv1_$T.log > gpurun_out/bench_mbv1_$T.json
python - <<PY
import json
for w in ("r50", "r8", "mbv1"):
    try:
        d = json.load(open(f"gpurun_out/bench_{w}_$T.json"))
        r = d["roofline"]
        print(w, d["value"], d.get("e2e", {}).get("value"), d.get("parity"), r["frac"],
              {k: (v.get("avg_us"), v.get("frac")) for k, v in r.get("kernels", {}).items()})
    except Exception as e:
        print(w, "ERR", e)
PY
