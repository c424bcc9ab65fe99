# launch list (durations) of the rasterizer bench section: build, accumulate, VJP kernels
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/raster_launches.csv python -c "
import sys,torch
sys.path.insert(0,'.')
import bench
bench.run_raster(torch, 2) if hasattr(bench,'run_raster') else None
" > gpurun_out/raster_launches.log 2>&1; echo "rc=$?" >> gpurun_out/raster_launches.log
