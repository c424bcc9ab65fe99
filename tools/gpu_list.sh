#!/bin/bash
# ncu launch list of a short bench run (run plain first by the box's ncu wrapper)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --grid-steps 1 --e2e-steps 1 \
  --stream-frames 50 --c5-iters 1 > gpurun_out/r_ncu_list.log 2>&1; echo "list rc=$?" >> gpurun_out/r_ncu_list.log
