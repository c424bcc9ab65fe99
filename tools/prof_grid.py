"""Profiling driver: C3 grid batches (for ncu runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
voxel = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
for _ in range(reps):
    gs = GridSampler(bench.GRID_INTR, voxel, occupied=VoxelHashSet(1 << 24))
    r = gs.sample(Dd, (Rd, Td), Cd)
torch.cuda.synchronize()
print("done", len(r))
