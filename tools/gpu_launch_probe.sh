cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
for pass in 1 2; do for m in torch direct; do
  timeout 600 python tools/stream_launch_probe.py $m >> gpurun_out/lp.log 2>&1
done; done
timeout 600 python tools/stream_host_split.py 300 >> gpurun_out/lp.log 2>&1
