#!/bin/bash
# Round evidence in one call: GPU tests, smoke, bench lines (r8 default with CPU baseline, r50, r62 sweep,
# reference arm), traffic + launch lists, ncu --set full of the ftable conv (r8 s0b0.a/b, r50 s0b1.b)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
TAG=${TAG:-full}
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3 | tee gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee gpurun_out/smoke_$TAG.txt
timeout 600 python bench.py 2>&1 | tail -1 | tee gpurun_out/bench_r8_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r8_$TAG.json --tuned-out gpurun_out/tuned_r8.json --report-out gpurun_out/report_r8_$TAG 2>&1 | tail -1 > gpurun_out/bench_r8_k20_$TAG.txt
timeout 900 python bench.py --workload r50 --steps 5 --warmup 3 --no-cpu-baseline --layers-out gpurun_out/layers_r50_$TAG.json --tuned-out gpurun_out/tuned_r50.json --report-out gpurun_out/report_r50_$TAG 2>&1 | tail -1 | tee gpurun_out/bench_r50_$TAG.txt
timeout 900 python bench.py --workload r62sweep --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r62sweep_$TAG.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_ref_$TAG.txt
TAG=$TAG bash scripts/gpu_ftprof.sh
