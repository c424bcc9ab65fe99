cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for c in 5 2; do
XGS_GRID_CSPLIT=$c timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_grid_async_gpu.py tests/test_shapes_gpu.py -k "grid or c3 or async" -q -x > gpurun_out/cs_tests_$c.log 2>&1; echo "rc=$?" >> gpurun_out/cs_tests_$c.log
done
for i in 1 2; do for c in 5 2 10; do XGS_GRID_CSPLIT=$c timeout 600 python tools/grid_bench.py 5 > gpurun_out/cs_${c}_$i.log 2>&1; done; done
