#!/bin/bash
# HEAD check: GPU tests, smoke, default bench line (ResNet-50 b256) and ResNet-8.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-f}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$T.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -4 gpurun_out/pytest_gpu_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1; tail -2 gpurun_out/smoke_$T.txt
timeout 900 python bench.py --steps 5 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$T.json --tuned-out gpurun_out/tuned_r50_$T.json > gpurun_out/bench_r50_$T.log 2>&1; tail -1 gpurun_out/bench_r50_$T.log > gpurun_out/bench_r50_$T.json
timeout 600 python bench.py --workload r8 --steps 20 --no-cpu-baseline --layers-out gpurun_out/layers_r8_$T.json --tuned-out gpurun_out/tuned_r8_$T.json > gpurun_out/bench_r8_$T.log 2>&1; tail -1 gpurun_out/bench_r8_$T.log > gpurun_out/bench_r8_$T.json
python - <<'PY'
import json,os
T=os.environ.get("TAG","f")
for w in ("r50","r8"):
    try:
        d=json.load(open(f"gpurun_out/bench_{w}_{T}.json"))
        print(w, d["value"], d["e2e"]["value"], d.get("parity",{}).get("status"), d["roofline"]["frac"], d["hbm"]["kernels"].get("quantize"))
    except Exception as e: print(w, "ERR", e)
PY
timeout 900 compute-sanitizer --tool racecheck --print-limit 40 python scripts/sanitize_cx.py > gpurun_out/racecheck_$T.txt 2>&1; grep -c "Race reported" gpurun_out/racecheck_$T.txt; grep -m6 -A3 "Race reported" gpurun_out/racecheck_$T.txt
