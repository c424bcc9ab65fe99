cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_thinker.py tests/test_raster.py -q -x > gpurun_out/th_tests.log 2>&1; echo "rc=$?" >> gpurun_out/th_tests.log
timeout 600 python -c "
import json,sys,torch
sys.path.insert(0,'.')
import bench
print(json.dumps(bench.run_consumers(torch, 5, cpu=False)))
" > gpurun_out/th_bench.log 2>&1
