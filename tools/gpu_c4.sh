cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in 1 2; do XGS_GRID_CSPLIT=$c timeout 900 python tools/stream_bench.py 1000 > gpurun_out/c4_cs$c.log 2>&1; done
timeout 900 python tools/stream_bench.py 1000 > gpurun_out/c4_default.log 2>&1
