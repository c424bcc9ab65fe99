"""Per-step host cost of GridSampler.sample's Python setup (C3 tensors)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200 import grid as g

D, C, R, T = bench.grid_scene()
Dd, Cd, Rd, Td = (torch.from_numpy(a).cuda() for a in (D, C, R, T))
N = 200


def tm(name, fn):
    fn()
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    print(f"{name:28s} {(time.perf_counter() - t0) / N * 1e6:7.1f} us")


tm("_dev(depth)", lambda: g._dev(Dd, torch.float32))
tm("_poses", lambda: g._poses((Rd, Td), 16))
tm("_dev(color)", lambda: g._dev(Cd, torch.uint8))
cap = 16 * 720 * 1280
tm("empty flat", lambda: torch.empty(11 * cap, dtype=torch.float64, device="cuda"))
tm("GridFrames", lambda: nat.GridFrames(16, 720, 1280, 1, 2, 3, 4, 1.0, 1.0, 1.0, 1.0, 0.01, 1, 0, 1e-3, None, 0, 0, 0))
tm("GridResult", lambda: nat.GridResult(cap, 1, 2, 3, 4, 5, 6, None, 7, 0, 0, 0, 0, 0))
tm("workspace", lambda: nat.workspace("grid", nat.lib().xgs_grid_workspace(cap)))
tm("stream_ptr", lambda: nat.stream_ptr())
tm("require_cuda", lambda: nat.require_cuda())
flat = torch.empty(11 * cap, dtype=torch.float64, device="cuda")
tm("7 views", lambda: (flat[:100].view(torch.int64), flat[cap:cap + 100].view(torch.int64), flat[2 * cap:2 * cap + 300].view(100, 3),
                       flat[5 * cap:5 * cap + 300].view(100, 3), flat[8 * cap:8 * cap + 100], flat[9 * cap:9 * cap + 100],
                       flat[10 * cap:10 * cap + 100]))
