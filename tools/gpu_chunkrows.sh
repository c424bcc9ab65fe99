cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for cr in 4194304 2097152 1048576; do XGS_SCREEN_CHUNK_ROWS=$cr timeout 900 python tools/c5_full.py 3 > gpurun_out/cr_$cr.log 2>&1; nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/cr_$cr.log; done
