"""GridSampler.sample on the C3 batch: host time in the Python wrapper vs inside the C-ABI call."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import cProfile
import pstats

import torch

import bench
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet

D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
hs = VoxelHashSet(bench.GRID_MAP + Dd.numel())
gs = GridSampler(bench.GRID_INTR, 0.01, occupied=hs)
inner = []
_call = nat.call


def call(name, *a):
    t0 = time.perf_counter()
    _call(name, *a)
    inner.append(time.perf_counter() - t0)


nat.call = call
tot = []
for i in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = gs.sample(Dd, (Rd, Td), Cd)
    tot.append(time.perf_counter() - t0)
print("sample() us median", np.median(tot[5:]) * 1e6, "inside nat.call", np.median(inner[5:]) * 1e6)
pr = cProfile.Profile()
pr.enable()
for i in range(20):
    gs.sample(Dd, (Rd, Td), Cd)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
