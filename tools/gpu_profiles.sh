#!/bin/bash
# Round profiles: launch list of a short default bench + full captures of the top kernels.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/p_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --grid-steps 1 --e2e-steps 1 \
  --stream-frames 50 > gpurun_out/p_list.log 2>&1; echo "list rc=$?" >> gpurun_out/p_list.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"screen_kernel" --launch-skip 40 -c 1 \
  -o gpurun_out/p_c5_screen python tools/prof_c5.py 1 > gpurun_out/p_c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/p_c5.log
XGS_WARM_FRAMES=32 timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:"grid_front_kernel|dd_scan_map|grid_pidlist_lb|grid_emit" --launch-skip 12 -c 4 \
  -o gpurun_out/p_grid python tools/prof_grid.py 2 0.01 > gpurun_out/p_grid.log 2>&1; echo "grid rc=$?" >> gpurun_out/p_grid.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_f64" -c 1 \
  -o gpurun_out/p_gemm python tools/prof_relevance.py 1 > gpurun_out/p_gemm.log 2>&1; echo "gemm rc=$?" >> gpurun_out/p_gemm.log
