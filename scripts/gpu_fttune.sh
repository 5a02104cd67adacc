#!/bin/bash
# ftable variant timings per layer (r8, r50 b64) + tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-ftt}
timeout 900 python -m pytest tests -q -m gpu -x ${PYTEST_K:-} 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python scripts/tune_variants.py --workload r8 --out gpurun_out/tune_r8_$TAG.json > gpurun_out/tune_r8_$TAG.log 2>&1
timeout 1200 python scripts/tune_variants.py --workload r50 --batch 64 --out gpurun_out/tune_r50_$TAG.json > gpurun_out/tune_r50_$TAG.log 2>&1
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi; true
