# C5 at N=1 with SMs reserved for the prep / accumulate streams while the screen runs
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for r in 0 16 8 24; do XGS_SCREEN_RESERVE_SMS=$r timeout 900 python tools/c5_full.py 3 > gpurun_out/c5res_$r.log 2>&1; done
