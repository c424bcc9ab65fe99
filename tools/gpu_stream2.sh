cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 600 python tools/stream_host.py 200 > gpurun_out/sh.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sh_launches.csv python tools/prof_stream.py 30 > gpurun_out/sh_ncu.log 2>&1
