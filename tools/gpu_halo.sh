cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for h in 1 0; do
XGS_GRID_HALO=$h timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_grid_async_gpu.py tests/test_shapes_gpu.py -k "grid or c3 or async" -q -x > gpurun_out/halo_tests_$h.log 2>&1; echo "rc=$?" >> gpurun_out/halo_tests_$h.log
done
for i in 1 2; do for h in 1 0; do XGS_GRID_HALO=$h timeout 600 python tools/grid_bench.py 5 > gpurun_out/halo_${h}_$i.log 2>&1; done; done
