#!/bin/bash
# One gpurun call: GPU parity tests, smoke, the default bench line (+ optional extra bench args).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-chk}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$TAG.txt
timeout ${TEST_TIMEOUT:-1200} python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu_$TAG.txt 2>&1
tail -30 gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1; tail -2 gpurun_out/smoke_$TAG.txt
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py ${BENCH:-} > gpurun_out/bench_$TAG.log 2>&1; tail -1 gpurun_out/bench_$TAG.log | tee gpurun_out/bench_$TAG.json
fi
