# ncu --set full of one fp64 contraction launch (relevance_per_gaussian, consumers bench)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_f64 -s 2 -c 1 \
  -o gpurun_out/dmma -f python -c "
import sys,torch
sys.path.insert(0,'.')
import bench
bench.run_consumers(torch, 1, cpu=False)
" > gpurun_out/ncu_dmma.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_dmma.log
