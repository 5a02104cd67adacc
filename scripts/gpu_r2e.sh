#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-e}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -8 gpurun_out/pytest_gpu_$T.txt
timeout 900 python bench.py --steps 5 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$T.json --tuned-out gpurun_out/tuned_r50_$T.json > gpurun_out/bench_r50_$T.log 2>&1; tail -1 gpurun_out/bench_r50_$T.log > gpurun_out/bench_r50_$T.json
timeout 900 python bench.py --workload mbv1 --steps 5 --no-cpu-baseline --layers-out gpurun_out/layers_mbv1_$T.json > gpurun_out/bench_mbv1_$T.log 2>&1; tail -1 gpurun_out/bench_mbv1_$T.log > gpurun_out/bench_mbv1_$T.json
python - <<'PY'
import json,os
T=os.environ.get("TAG","e")
for w in ("r50","mbv1"):
    try:
        d=json.load(open(f"gpurun_out/bench_{w}_{T}.json"))
        print(w, d["value"], d.get("parity",{}).get("status"), d["roofline"]["frac"], {k:(v["avg_us"],v["glookup_s"]) for k,v in d["roofline"]["kernels"].items()})
    except Exception as e: print(w, "ERR", e)
PY
