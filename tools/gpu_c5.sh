cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=memory.total,memory.used --format=csv > gpurun_out/c5_mem.log 2>&1
timeout 900 python -m pytest tests/test_vq_chunks_gpu.py tests/test_vq_gpu.py -q -x > gpurun_out/c5_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c5_tests.log
timeout 900 python tools/c5_full.py 3 > gpurun_out/c5_full.log 2>&1; echo "rc=$?" >> gpurun_out/c5_full.log
