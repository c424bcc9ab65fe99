# C4 launch list: every kernel of ~60 stream frames (graph kernel nodes profiled one by one),
# durations only; the per-frame graph body is read off the steady-state frames.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/c4_launches.csv python tools/stream_bench.py 60 > gpurun_out/c4_launches.log 2>&1
echo "rc=$?" >> gpurun_out/c4_launches.log
