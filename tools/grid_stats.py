"""Item / voxel counts of one C3 batch (how much the front-end dedup leaves to the sort)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet
D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
for v in (0.01, 0.05):
    gs = GridSampler(bench.GRID_INTR, v, occupied=VoxelHashSet(1 << 24))
    r = gs.sample(Dd, (Rd, Td), Cd)
    print(v, "valid", r.n_valid, "sorted", r.n_sorted, "voxels", r.n_voxels, "new", len(r), "passes", r.sort_passes)
