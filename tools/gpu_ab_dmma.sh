# A/B of decode_f64.cu variants (tools/ab/decode_f64_<tag>.cu): thinker tests + the consumers bench
cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out
SRC=paper_2603_09632_b200/csrc/decode_f64.cu
cp $SRC /tmp/dec_orig.cu
for pass in 1 2; do for v in tools/ab/decode_f64_*.cu; do
  tag=$(basename $v .cu); tag=${tag#decode_f64_}
  cp $v $SRC
  python -c "from paper_2603_09632_b200 import build as b; b.build()" > gpurun_out/abd_build_$tag.log 2>&1
  if [ $pass = 1 ]; then
    timeout 900 python -m pytest tests/test_thinker.py -q -x > gpurun_out/abd_tests_$tag.log 2>&1; echo "rc=$?" >> gpurun_out/abd_tests_$tag.log
  fi
  timeout 600 python -c "
import json,sys,torch
sys.path.insert(0,'.')
import bench
r = bench.run_consumers(torch, 5, cpu=False)['relevance_per_gaussian']
print('$tag', $pass, round(r['ms'], 2), round(r['fp64_frac'], 3))
" >> gpurun_out/abd_bench.log 2>&1
done; done
cp /tmp/dec_orig.cu $SRC
