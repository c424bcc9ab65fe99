"""Host-side cost of GridSampler.sample at C3 (1 cm): the Python setup before
the native call, the native call (two read-back syncs inside), the result
wrap-up; device time from CUDA events for comparison."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet, pack_key

D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
rng = np.random.default_rng(22)
pts = rng.uniform(-4.0, 4.0, (bench.GRID_MAP, 3))
q = np.floor(pts / 0.01).astype(np.int64)
warm = torch.from_numpy(pack_key(q[:, 0], q[:, 1], q[:, 2]).view(np.int64)).cuda()
orig = nat.call
marks = {}


def call(name, *a):
    if name == "xgs_grid_sample":
        marks["call0"] = time.perf_counter()
        r = orig(name, *a)
        marks["call1"] = time.perf_counter()
        return r
    return orig(name, *a)


nat.call = call
import paper_2603_09632_b200.grid as g
g.nat.call = call
rows = []
r = None
for it in range(8):
    hs = VoxelHashSet(bench.GRID_MAP + bench.GRID_F * bench.GRID_H * bench.GRID_W)
    hs.insert(warm)
    gs = GridSampler(bench.GRID_INTR, 0.01, occupied=hs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    r = gs.sample(Dd, (Rd, Td), Cd)
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    rows.append(((marks["call0"] - t0) * 1e3, (marks["call1"] - marks["call0"]) * 1e3, (t1 - marks["call1"]) * 1e3,
                 e0.elapsed_time(e1)))
    hs.close()
a = np.array(rows[2:])
print("setup ms %.3f  native call ms %.3f  wrap ms %.3f  events ms %.3f" % tuple(np.median(a, axis=0)))

import cProfile
import pstats
nat.call = orig
g.nat.call = orig
hs = VoxelHashSet(bench.GRID_MAP + bench.GRID_F * bench.GRID_H * bench.GRID_W)
hs.insert(warm)
gs = GridSampler(bench.GRID_INTR, 0.01, occupied=hs)
for _ in range(3):
    r = gs.sample(Dd, (Rd, Td), Cd)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    r = gs.sample(Dd, (Rd, Td), Cd)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
