cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_grid_async_gpu.py tests/test_stream_gpu.py -q -x > gpurun_out/ft_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ft_tests.log
XGS_GRID_SORT=1 timeout 900 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/ft_tests_sort.log 2>&1; echo "rc=$?" >> gpurun_out/ft_tests_sort.log
for i in 1 2; do timeout 900 python tools/stream_bench.py 1000 > gpurun_out/ft_bench_$i.log 2>&1; done
