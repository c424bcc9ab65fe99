# ncu --set full of the table scan (C3 1 cm and 5 cm, GridGraph replay after a map restore)
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export XGS_WARM_FRAMES=60
for v in 0.01 0.05; do
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:dd_scan -s 2 -c 1 \
  -o gpurun_out/scan_$v -f python tools/grid_graph_once.py $v 3 > gpurun_out/ncu_scan_$v.log 2>&1
done
