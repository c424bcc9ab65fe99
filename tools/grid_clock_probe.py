"""Is the C3 grid batch slower in isolation than back to back?  GridGraph
replays of the 1 cm batch timed (a) after a map restore + host sync, (b) the
same with a ~2 ms busy GEMM queued right before the replay, (c) 10 replays
back to back (map not restored: later replays find no new voxels)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet

D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
voxel = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
warm, _, _ = bench.grid_warm_map(torch, voxel, max_frames=int(os.environ.get("XGS_WARM_FRAMES", "240")))
npix = Dd.numel()
snap = VoxelHashSet(bench.GRID_MAP + npix)
snap.insert(warm)
work = VoxelHashSet(bench.GRID_MAP + npix)
work.copy_from(snap)
gg = GridGraph(GridSampler(bench.GRID_INTR, voxel, occupied=work), Dd, (Rd, Td), Cd)
A = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)


def timed(busy):
    work.copy_from(snap)
    torch.cuda.synchronize()
    if busy:
        for _ in range(4):
            A @ A
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gg.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for busy in (False, True, False, True):
    ts = [timed(busy) for _ in range(8)]
    print("busy" if busy else "idle", "median ms", round(float(np.median(ts[1:])), 4), [round(x, 4) for x in ts])
work.copy_from(snap)
torch.cuda.synchronize()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
evs[0].record()
for i in range(10):
    gg.replay()
    evs[i + 1].record()
torch.cuda.synchronize()
print("back-to-back", [round(evs[i].elapsed_time(evs[i + 1]), 4) for i in range(10)])
clk = bench.ClockSampler(0)
clk.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(3000):
    gg.replay()
e1.record()
torch.cuda.synchronize()
print("3000 back-to-back: ms per replay", round(e0.elapsed_time(e1) / 3000, 4), "clocks", clk.stop())
