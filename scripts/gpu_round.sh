#!/bin/bash
# One gpurun call: device info, GPU parity tests, a short bench.  Outputs land in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv | tee gpurun_out/smi.txt
python -c "import torch; p=torch.cuda.get_device_properties(0); print(p, p.multi_processor_count)" 2>&1 | tail -2
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -q -m gpu ${PYTEST_ARGS:-} 2>&1 | tail -40 | tee gpurun_out/pytest_gpu.txt
if [ -n "$BENCH" ]; then
  timeout 600 python bench.py $BENCH 2>&1 | tail -5 | tee gpurun_out/bench.txt
fi
