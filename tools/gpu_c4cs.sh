cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in 1 5; do for i in 1 2; do XGS_GRID_CSPLIT=$c timeout 900 python tools/stream_bench.py 1000 > gpurun_out/c4cs_${c}_$i.log 2>&1; done; done
XGS_GRID_CSPLIT=5 timeout 900 python -m pytest tests/test_stream_gpu.py tests/test_grid_gpu.py -q -x > gpurun_out/c4cs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c4cs_tests.log
