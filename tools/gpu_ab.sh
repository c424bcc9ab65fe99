# A/B of grid.cu variants: tools/ab/grid_<tag>.cu each built into the library in turn
# (ROUNDS passes, alternating), grid parity tests on the first pass, tools/grid_bench.py every pass
# (STREAM=1: tools/stream_bench.py too).
# The variant files are scratch (not committed); the working grid.cu is restored at the end.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
SRC=paper_2603_09632_b200/csrc/grid.cu
cp $SRC /tmp/grid_orig.cu
for pass in $(seq 1 ${ROUNDS:-2}); do
  for v in tools/ab/grid_*.cu; do
    tag=$(basename $v .cu); tag=${tag#grid_}
    cp $v $SRC
    python -c "from paper_2603_09632_b200 import build as b; b.build()" > gpurun_out/ab_build_$tag.log 2>&1
    if [ $pass = 1 ]; then
      timeout 900 python -m pytest tests/test_grid_gpu.py tests/test_grid_async_gpu.py tests/test_stream_gpu.py -q -x > gpurun_out/ab_tests_$tag.log 2>&1
      echo "rc=$?" >> gpurun_out/ab_tests_$tag.log
    fi
    timeout 600 python tools/grid_bench.py 5 > gpurun_out/ab_${tag}_$pass.log 2>&1
    if [ -n "$STREAM" ]; then timeout 600 python tools/stream_bench.py 1000 > gpurun_out/abs_${tag}_$pass.log 2>&1; fi
  done
done
cp /tmp/grid_orig.cu $SRC
