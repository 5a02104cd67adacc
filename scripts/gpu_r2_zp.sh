cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
./build/lds128_quarters | tee gpurun_out/lds128_quarters.json
timeout 600 python scripts/zp_stats.py --workload r50 --images 2 --out gpurun_out/zp_r50.json > gpurun_out/zp_r50.log 2>&1; tail -3 gpurun_out/zp_r50.log
timeout 300 python scripts/zp_stats.py --workload r8 --images 64 --out gpurun_out/zp_r8.json > gpurun_out/zp_r8.log 2>&1; tail -3 gpurun_out/zp_r8.log
