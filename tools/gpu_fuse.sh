cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2 3; do for f in 1 0; do XGS_GRID_FUSE_EMIT=$f timeout 600 python tools/grid_bench.py 5 > gpurun_out/fu_${f}_$i.log 2>&1; done; done
