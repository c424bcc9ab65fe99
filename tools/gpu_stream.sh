cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_stream_gpu.py tests/test_grid_gpu.py -q -x > gpurun_out/s_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s_tests.log
timeout 900 python tools/stream_bench.py 1000 > gpurun_out/s_bench.log 2>&1; echo "rc=$?" >> gpurun_out/s_bench.log
