"""Host-side profile of GridSampler.sample on the C3 1 cm batch: wall time per call vs the
device span, and cProfile of 200 calls (the map is not restored between calls: after the first
call nearly every voxel is old, which does not change the host work)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet

D, C, R, T = bench.grid_scene()
Dd, Cd = torch.from_numpy(D).cuda(), torch.from_numpy(C).cuda()
Rd, Td = torch.from_numpy(R).cuda(), torch.from_numpy(T).cuda()
hs = VoxelHashSet(bench.GRID_MAP_SLOTS)
gs = GridSampler(bench.GRID_INTR, 0.01, occupied=hs)
for _ in range(5):
    gs.sample(Dd, (Rd, Td), Cd)
torch.cuda.synchronize()
ts = []
for _ in range(50):
    t0 = time.perf_counter()
    r = gs.sample(Dd, (Rd, Td), Cd)
    ts.append(time.perf_counter() - t0)
print("wall per call (median, us):", round(np.median(ts) * 1e6, 1))
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    gs.sample(Dd, (Rd, Td), Cd)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
