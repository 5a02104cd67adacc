#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 3 --layers-out gpurun_out/layers_r8_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r8_$TAG.txt
timeout 900 python bench.py --workload r50 --steps 3 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r50_$TAG.txt
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi; true
