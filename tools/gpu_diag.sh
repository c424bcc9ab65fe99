# A/B of the front end's dedup width (XGS_GRID_DIAG 0/1/2; no rebuild), two passes
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for pass in 1 2; do for dg in 2 1 0; do
  XGS_GRID_DIAG=$dg timeout 600 python tools/grid_bench.py 5 > gpurun_out/ab_diag${dg}_$pass.log 2>&1
done; done
