# ncu --set full of the two hashed front ends (block vs persistent) on C3 1 cm, warm map of 60 frames
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
export XGS_WARM_FRAMES=60
XGS_GRID_FRONT=block timeout 900 ncu --set full --import-source on --clock-control none -k regex:grid_front -s 1 -c 1 \
  -o gpurun_out/front_block -f python tools/prof_grid.py 2 0.01 > gpurun_out/ncu_front_block.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:grid_front -s 1 -c 1 \
  -o gpurun_out/front_pers -f python tools/prof_grid.py 2 0.01 > gpurun_out/ncu_front_pers.log 2>&1
