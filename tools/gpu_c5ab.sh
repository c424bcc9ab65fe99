cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for e in 0 1; do XGS_SCREEN_PF_EARLY=$e timeout 900 python tools/c5_full.py 6 > gpurun_out/c5ab_$e.log 2>&1; done
XGS_SCREEN_PF_EARLY=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:screen_kernel --launch-skip 32 -c 32 --csv --log-file gpurun_out/c5ab_ncu.csv python tools/prof_c5.py 1 > gpurun_out/c5ab_ncu.log 2>&1
timeout 600 python -m pytest tests/test_vq_gpu.py tests/test_shapes_gpu.py -q -x -k "c5 or assign or online" > gpurun_out/c5ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c5ab_tests.log
