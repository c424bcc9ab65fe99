cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
timeout 300 python tools/grid_bench.py 5 > gpurun_out/g_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g_bench.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"grid_front" -c 2 -o gpurun_out/g_front python tools/prof_grid.py 1 0.01 > gpurun_out/g_ncu.log 2>&1; echo "rc=$?" >> gpurun_out/g_ncu.log
