"""One C3 batch through GridGraph after a map restore (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet

D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
voxel = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
warm, _, _ = bench.grid_warm_map(torch, voxel, max_frames=int(os.environ.get("XGS_WARM_FRAMES", "60")))
npix = Dd.numel()
snap = VoxelHashSet(bench.GRID_MAP + npix)
snap.insert(warm)
work = VoxelHashSet(bench.GRID_MAP + npix)
work.copy_from(snap)
gg = GridGraph(GridSampler(bench.GRID_INTR, voxel, occupied=work), Dd, (Rd, Td), Cd)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("replays")
for _ in range(reps):
    work.copy_from(snap)
    gg.replay()
    torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done", len(gg.result()))
