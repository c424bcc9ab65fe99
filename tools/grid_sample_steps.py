"""Host-time of each step inside GridSampler.sample (C3 tensors, warm), to find
the Python overhead around the native call."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200 import grid as g

D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
hs = g.VoxelHashSet(1 << 25)
gs = g.GridSampler(bench.GRID_INTR, 0.05, occupied=hs)
for _ in range(3):
    r = gs.sample(Dd, (Rd, Td), Cd)
torch.cuda.synchronize()
acc = {}


def mark(name, t0):
    t1 = time.perf_counter()
    acc.setdefault(name, []).append((t1 - t0) * 1e6)
    return t1


t = torch
for it in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d = g._dev(Dd, t.float32); t0 = mark("dev depth", t0)
    F, H, W = (int(v) for v in d.shape); t0 = mark("shape", t0)
    Rr, tr = g._poses((Rd, Td), F); t0 = mark("poses", t0)
    col = g._dev(Cd, t.uint8); t0 = mark("dev color", t0)
    cap = F * H * W
    flat = t.empty(11 * cap, dtype=t.float64, device="cuda"); t0 = mark("empty", t0)
    b = flat.data_ptr()
    fx, fy, cx, cy = gs.intr
    fr = nat.GridFrames(F, H, W, d.data_ptr(), col.data_ptr(), Rr.data_ptr(), tr.data_ptr(), fx, fy, cx, cy, gs.voxel, 1,
                        0, gs.min_scale, None, 0, 0, 0); t0 = mark("frames struct", t0)
    res = nat.GridResult(cap, b, b + 8 * cap, b + 16 * cap, b + 40 * cap, b + 64 * cap, b + 72 * cap, None,
                         b + 80 * cap, 0, 0, 0, 0, 0, 0); t0 = mark("result struct", t0)
    ws = nat.workspace("grid", nat.lib().xgs_grid_workspace(F * H * W)); t0 = mark("workspace", t0)
    sp = nat.stream_ptr(); t0 = mark("stream_ptr", t0)
    nat.call("xgs_grid_sample", ctypes.byref(fr), hs._h, ctypes.byref(res), nat.ptr(ws), ws.numel(), sp)
    t0 = mark("native call", t0)
    n = int(res.n_new)
    out = g.GridSampleResult(flat, cap, n, None, int(res.n_valid), int(res.n_voxels), int(res.n_sorted),
                             int(res.sort_passes)); t0 = mark("wrap", t0)
for k, v in acc.items():
    print(f"{k:16s} {np.median(v[5:]):8.1f} us")
