# accumulate_dev parity + stream tests, then the stream bench twice
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_vq_gpu.py tests/test_stream_gpu.py tests/test_distributed_cpu.py -q -x > gpurun_out/ad_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ad_tests.log
for i in 1 2; do timeout 600 python tools/stream_bench.py 1000 > gpurun_out/ad_bench_$i.log 2>&1; done
