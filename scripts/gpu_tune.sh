#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-t1}
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -25 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 900 python scripts/tune_variants.py --workload r8 --out gpurun_out/tune_r8_$TAG.json 2>&1 | tail -3
timeout 1200 python scripts/tune_variants.py --workload r50 --batch 64 --out gpurun_out/tune_r50_$TAG.json 2>&1 | tail -3
timeout 600 python bench.py --steps 20 --warmup 3 --layers-out gpurun_out/layers_r8_$TAG.json 2>&1 | tail -1 | tee gpurun_out/bench_r8_$TAG.txt
