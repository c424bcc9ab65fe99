# C4 stream bench under each front-end dedup width (XGS_GRID_DIAG; no rebuild)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for pass in 1 2; do for dg in 2 1 0; do
  XGS_GRID_DIAG=$dg timeout 600 python tools/stream_bench.py 1000 > gpurun_out/abs_diag${dg}_$pass.log 2>&1
done; done
