cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
run() { env "$@" timeout 600 python tools/grid_bench.py 5 > gpurun_out/tb_$(echo "$@" | tr ' =' '_-').log 2>&1; }
for scan in loads bulk; do
run XGS_GRID_SCAN=$scan XGS_GRID_TABLE_SLACK=2
run XGS_GRID_SCAN=$scan XGS_GRID_TABLE_SLACK=1
run XGS_GRID_SCAN=$scan XGS_GRID_TABLE_SLACK=1 XGS_GRID_TABLE_FACTOR=2
run XGS_GRID_SCAN=$scan XGS_GRID_TABLE_SLACK=1 XGS_GRID_TABLE_MIN=65536
run XGS_GRID_SCAN=$scan XGS_GRID_TABLE_SLACK=1 XGS_GRID_TABLE_FACTOR=2 XGS_GRID_TABLE_MIN=65536
done
