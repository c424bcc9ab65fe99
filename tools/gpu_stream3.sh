cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_stream_gpu.py -q -x > gpurun_out/s3_tests.log 2>&1; echo "rc=$?" >> gpurun_out/s3_tests.log
timeout 600 python tools/stream_host.py 1000 > gpurun_out/s3.log 2>&1
