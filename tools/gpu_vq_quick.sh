#!/bin/bash
# VQ + grid GPU tests and a short default bench (no CPU leg, shorter stream), for quick confirmation runs.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/q_tests.log 2>&1; echo "rc=$?" >> gpurun_out/q_tests.log
timeout 900 python bench.py --no-cpu > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "rc=$?" >> gpurun_out/q_bench.err
