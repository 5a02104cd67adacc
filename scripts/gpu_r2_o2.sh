#!/bin/bash
# The two-CTAs-per-SM CX variant: GPU tests (every variant vs the oracle), then the ResNet-50 / ResNet-8 steps
# autotuned with it available vs the previous picks (build/tuned_*.json), per-layer tables.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_o2.txt 2>&1; tail -2 gpurun_out/pytest_o2.txt
for w in r50 r8; do
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --tuned-out gpurun_out/tuned_o2_$w.json \
    --layers-out gpurun_out/layers_o2_$w.json > gpurun_out/bench_o2_$w.log 2>&1
  timeout 600 python bench.py --workload $w --steps 5 --no-cpu-baseline --tuned-from build/tuned_$w.json \
    --layers-out gpurun_out/layers_o2old_$w.json > gpurun_out/bench_o2old_$w.log 2>&1
  for t in o2 o2old; do
    python -c "import json; d=json.loads(open('gpurun_out/bench_${t}_$w.log').read().strip().splitlines()[-1]); print('$w $t', d['value'], d['parity']['status'], d['roofline']['frac'])"
  done
done
python - <<'PY'
import json
for w in ("r50", "r8"):
    try:
        a = json.load(open(f"gpurun_out/layers_o2_{w}.json")); b = json.load(open(f"gpurun_out/layers_o2old_{w}.json"))
        for x, y in zip(a, b):
            if x["variant"] != y["variant"]:
                print(w, x["node"], x["variant"], x["ms"], "vs", y["variant"], y["ms"])
    except Exception as e:
        print(w, "ERR", e)
PY
