cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv python tools/prof_c5.py 2 > gpurun_out/c5_list.log 2>&1; echo "rc=$?" >> gpurun_out/c5_list.log
