cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_vq_gpu.py tests/test_vq_chunks_gpu.py tests/test_shapes_gpu.py tests/test_stream_gpu.py tests/test_multirank_gpu.py -q -x > gpurun_out/rr_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rr_tests.log
for i in 1 2; do timeout 900 python tools/c5_full.py 3 > gpurun_out/rr_c5_$i.log 2>&1; done
