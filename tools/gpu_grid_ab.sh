cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
XGS_GRID_SPLIT_INSERT=1 timeout 600 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
for si in 0 1 0 1; do XGS_GRID_SPLIT_INSERT=$si timeout 600 python tools/grid_bench.py 5 >> gpurun_out/g_bench_$si.log 2>&1; done
