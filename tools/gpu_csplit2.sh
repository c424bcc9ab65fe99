# C3 front-end blocks per row band (XGS_GRID_CSPLIT, no rebuild), two passes
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for pass in 1 2; do for cs in 2 1 5; do
  XGS_GRID_CSPLIT=$cs timeout 600 python tools/grid_bench.py 5 > gpurun_out/ab_cs${cs}_$pass.log 2>&1
done; done
