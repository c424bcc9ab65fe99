cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_native_abi.py tests/test_vq_gpu.py -q -x > gpurun_out/sr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sr_tests.log
timeout 900 python tools/stream_host_split.py 300 > gpurun_out/sr_split.log 2>&1
for i in 1 2; do timeout 900 python tools/stream_bench.py 1000 > gpurun_out/sr_bench_$i.log 2>&1; done
