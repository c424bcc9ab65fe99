#!/bin/bash
# GPU test suite + smoke (quick confirmation pass).
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 ${TESTS:-} > gpurun_out/t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/t_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/t_smoke.log
