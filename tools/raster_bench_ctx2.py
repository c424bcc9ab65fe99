"""bench.run_raster after a 150 GB allocation was freed (the C5 headline's footprint)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
r = bench.run_raster(torch, 3, cpu=False)
print("alone", r["build_ms"], r["vjp_ms"])
big = torch.empty(150 * 2**30, dtype=torch.uint8, device="cuda")
big.fill_(1)
del big
torch.cuda.empty_cache()
r = bench.run_raster(torch, 3, cpu=False)
print("after 150 GB alloc/free", r["build_ms"], r["vjp_ms"])
r = bench.run_raster(torch, 3, cpu=False)
print("again", r["build_ms"], r["vjp_ms"])
