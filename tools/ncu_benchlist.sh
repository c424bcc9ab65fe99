# launch list (per-kernel duration + DRAM bytes) of a short default-shaped bench run (C5 headline, C2, C4
# stream); the grid batch has its own lists (tools/ncu_grid3.sh)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/p6_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-grid --e2e-steps 1 \
  --stream-frames 50 > gpurun_out/p6_list.log 2>&1; echo "list rc=$?" >> gpurun_out/p6_list.log
