"""Profiling driver: C3 grid batches against the scene-derived running map (bench.run_grid's setup), for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
voxel = float(sys.argv[2]) if len(sys.argv) > 2 else 0.01
D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
warm, _, _ = bench.grid_warm_map(torch, voxel, max_frames=int(os.environ.get("XGS_WARM_FRAMES", "240")))
npix = bench.GRID_F * bench.GRID_H * bench.GRID_W
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
for _ in range(reps):
    hs = VoxelHashSet(bench.GRID_MAP + npix)
    hs.insert(warm)
    gs = GridSampler(bench.GRID_INTR, voxel, occupied=hs)
    r = gs.sample(Dd, (Rd, Td), Cd)
    torch.cuda.synchronize()
    hs.close()
torch.cuda.nvtx.range_pop()
print("done", len(r))
