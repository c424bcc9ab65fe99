cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"grid_front_kernel|dd_scan_map|grid_pidlist_lb" --launch-skip 3 -c 3 -o gpurun_out/g_full python tools/prof_grid.py 3 0.01 > gpurun_out/g_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/g_ncu.log
