cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for i in 1 2; do for pr in 1 0; do XGS_PIPE_PRIO=$pr timeout 900 python tools/c5_full.py 3 > gpurun_out/pr_${pr}_$i.log 2>&1; done; done
