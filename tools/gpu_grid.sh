cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
timeout 300 python tools/grid_bench.py 5 > gpurun_out/g_bench.log 2>&1; echo "rc=$?" >> gpurun_out/g_bench.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/g_launches.csv python tools/prof_grid.py 1 0.01 > gpurun_out/g_list.log 2>&1; echo "rc=$?" >> gpurun_out/g_list.log
