"""Profiling driver: the bench's rasterizer scene (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
print(bench.run_raster(torch, int(sys.argv[1]) if len(sys.argv) > 1 else 1, cpu=False))
