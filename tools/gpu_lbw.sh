cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_grid_async_gpu.py tests/test_stream_gpu.py tests/test_shapes_gpu.py -k "grid or c3 or async or stream" -q -x > gpurun_out/lbw_tests.log 2>&1; echo "rc=$?" >> gpurun_out/lbw_tests.log
XGS_GRID_SORT=1 timeout 900 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/lbw_tests_sort.log 2>&1; echo "rc=$?" >> gpurun_out/lbw_tests_sort.log
for i in 1 2; do timeout 900 python tools/stream_bench.py 1000 > gpurun_out/lbw_c4_$i.log 2>&1; done
timeout 600 python tools/grid_bench.py 5 > gpurun_out/lbw_c3.log 2>&1
