# Grid evidence (round 2, session 3): full captures of the C3 1 cm batch's kernels (GridGraph replay
# after a map restore) + their launch list with DRAM bytes, both voxel sizes.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export XGS_WARM_FRAMES=60
timeout 900 ncu --set full --import-source on --clock-control none \
  -k regex:"grid_front_kernel|dd_scan_map|grid_pidlist_lb" -s 6 -c 3 \
  -o gpurun_out/p_grid3 -f python tools/grid_graph_once.py 0.01 3 > gpurun_out/p_grid3.log 2>&1; echo "rc=$?" >> gpurun_out/p_grid3.log
for v in 0.01 0.05; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"grid_front_kernel|dd_scan_map|grid_pidlist_lb|grid_emit" --csv --log-file gpurun_out/p_grid3_list_$v.csv \
  python tools/grid_graph_once.py $v 3 > gpurun_out/p_grid3_list_$v.log 2>&1
done
