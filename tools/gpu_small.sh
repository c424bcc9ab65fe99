cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_vq_gpu.py tests/test_stream_gpu.py tests/test_shapes_gpu.py tests/test_vq_chunks_gpu.py -q -x > gpurun_out/sm_tests.log 2>&1; echo "rc=$?" >> gpurun_out/sm_tests.log
for v in 0 16384; do for i in 1 2; do XGS_SCREEN_SMALL_ROWS=$v timeout 900 python tools/stream_bench.py 1000 > gpurun_out/sm_bench_${v}_$i.log 2>&1; done; done
