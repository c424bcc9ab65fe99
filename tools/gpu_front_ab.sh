cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_grid_async_gpu.py tests/test_shapes_gpu.py -k "grid or c3 or async" -q -x > gpurun_out/fab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fab_tests.log
XGS_GRID_SORT=1 timeout 900 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/fab_tests_sort.log 2>&1; echo "rc=$?" >> gpurun_out/fab_tests_sort.log
for i in 1 2 3; do timeout 600 python tools/grid_bench.py 5 > gpurun_out/fab_$i.log 2>&1; done
