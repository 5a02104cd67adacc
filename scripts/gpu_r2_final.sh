#!/bin/bash
# Final HEAD check, the driver's own commands: GPU tests, smoke, `bench.py --gpus 1 --steps 20 --warmup 5`,
# the reference arm, and the config-5 exact-LUT control on the ResNet-50 shape (--lut exact).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-final}
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_$T.txt 2>&1; tail -2 gpurun_out/pytest_gpu_$T.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.txt 2>&1; tail -1 gpurun_out/smoke_$T.txt
S=$SECONDS; timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_r50_$T.log 2> gpurun_out/bench_r50_$T.err; echo "bench wall $((SECONDS-S)) s"
tail -1 gpurun_out/bench_r50_$T.log > gpurun_out/bench_r50_$T.json
S=$SECONDS; timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_$T.log 2> gpurun_out/bench_ref_$T.err; echo "reference arm wall $((SECONDS-S)) s"
tail -1 gpurun_out/bench_ref_$T.log > gpurun_out/bench_ref_$T.json
timeout 900 python bench.py --lut exact --steps 10 --no-cpu-baseline > gpurun_out/bench_r50exact_$T.log 2>&1
tail -1 gpurun_out/bench_r50exact_$T.log > gpurun_out/bench_r50exact_$T.json
python - <<PY
import json
for w in ("r50", "ref", "r50exact"):
    d = json.load(open(f"gpurun_out/bench_{w}_$T.json"))
    print(w, d["value"], d["e2e"]["value"], d.get("parity", {}).get("status") if isinstance(d.get("parity"), dict) else None,
          d.get("roofline", {}).get("frac"), d["config"].get("lut"), d.get("clocks", {}).get("reasons"))
PY
