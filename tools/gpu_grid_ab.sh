cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
for i in 1 2; do timeout 600 python tools/grid_bench.py 5 >> gpurun_out/g_bench.log 2>&1; done
