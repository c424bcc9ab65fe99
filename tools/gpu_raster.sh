# rasterizer parity tests + the raster bench section
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_raster.py tests/test_thinker.py -q -x > gpurun_out/rs_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rs_tests.log
timeout 600 python -c "
import json,sys,torch
sys.path.insert(0,'.')
import bench, gc
gc.disable()
r = bench.run_raster(torch, 7, cpu=False)
print(json.dumps({k: r[k] for k in ('build_ms','accumulate_ms','vjp_ms','pairs')}))
" > gpurun_out/rs_bench.log 2>&1
