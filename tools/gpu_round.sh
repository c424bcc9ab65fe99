#!/bin/bash
# One GPU pass: tests, smoke, default bench, ncu launch list + full captures of the top kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r_smoke.log
timeout 900 python bench.py > gpurun_out/r_bench.json 2> gpurun_out/r_bench.err; echo "bench rc=$?" >> gpurun_out/r_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --grid-steps 1 --e2e-steps 1 \
  --stream-frames 50 --c5-iters 1 > gpurun_out/r_ncu_list.log 2>&1; echo "list rc=$?" >> gpurun_out/r_ncu_list.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"screen_kernel|prep_rows|acc_chain" -c 4 \
  -o gpurun_out/r_vq_full python tools/prof_vq.py 2 > gpurun_out/r_ncu_vq.log 2>&1; echo "vq rc=$?" >> gpurun_out/r_ncu_vq.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"grid_front|dd_insert|dd_scan|grid_emit|grid_pidlist" -c 5 \
  -o gpurun_out/r_grid_full python tools/prof_grid.py 1 0.01 > gpurun_out/r_ncu_grid.log 2>&1; echo "grid rc=$?" >> gpurun_out/r_ncu_grid.log
