# A/B of the front end's rows per block (FK_ROWS): rebuilds the library with each value in turn
# (sed on a copy of grid.cu), runs the grid bench + grid parity tests, restores the source.
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
SRC=paper_2603_09632_b200/csrc/grid.cu
cp $SRC /tmp/grid_orig.cu
for fk in ${FK_LIST:-4 5 6 7}; do
  sed "s/^constexpr int FK_ROWS = [0-9]*;/constexpr int FK_ROWS = $fk;/; s/kFrontBlocksPerSM = FK_ROWS <= 6 ? 3 : 2;/kFrontBlocksPerSM = 3;/" \
    /tmp/grid_orig.cu > $SRC
  python -c "from paper_2603_09632_b200 import build as b; b.build()" > gpurun_out/fk_build_$fk.log 2>&1
  timeout 600 python tools/grid_bench.py 5 > gpurun_out/fk_$fk.log 2>&1
  timeout 600 python -m pytest tests/test_grid_gpu.py -q -x > gpurun_out/fk_tests_$fk.log 2>&1; echo "rc=$?" >> gpurun_out/fk_tests_$fk.log
done
cp /tmp/grid_orig.cu $SRC
python -c "from paper_2603_09632_b200 import build as b; b.build()" > gpurun_out/fk_build_final.log 2>&1
