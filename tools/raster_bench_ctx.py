"""bench.run_raster alone, then after the other sub-benchmarks that precede it in bench.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
r = bench.run_raster(torch, 3, cpu=False)
print("alone", r["build_ms"], r["vjp_ms"], r["accumulate_ms"])
bench.run_targets(torch, 10, cpu=False)
bench.run_init(torch, cpu=False)
bench.run_consumers(torch, 5, cpu=False)
r = bench.run_raster(torch, 3, cpu=False)
print("after targets/init/consumers", r["build_ms"], r["vjp_ms"], r["accumulate_ms"])
