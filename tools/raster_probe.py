"""Rasterizer build: host wall time of the C call vs the whole _Pairs construction (profiling aid)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200 import rasterizer as rz
from paper_2603_09632_b200.core import CameraIntrinsics, CameraPose
from paper_2603_09632_b200.supervision import GridSpec

n, H, W, s = 1 << 18, 480, 640, 4
g = torch.Generator(device="cuda")
g.manual_seed(70)
z = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 7.0 + 0.5
u = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5) * z * (H / 525.0)
v = (torch.rand(n, generator=g, device="cuda", dtype=torch.float64) - 0.5) * z * (W / 525.0)
q = torch.randn(n, 4, generator=g, device="cuda", dtype=torch.float64)
field = type("DeviceField", (), {
    "mu": torch.stack([u, v, z], 1).contiguous(), "quat": (q / q.norm(dim=1, keepdim=True)).contiguous(),
    "scale": torch.exp(torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64) * 2.3 - 4.6),
    "opacity": torch.rand(n, generator=g, device="cuda", dtype=torch.float64) * 0.9 + 0.05,
    "color": torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64),
    "__len__": lambda self: n})()
intr = CameraIntrinsics(fx=525.0, fy=525.0, cx=239.5, cy=319.5, height=H, width=W)
pose = CameraPose.identity()
grid = GridSpec(H=H, W=W, s=s)
inner = []
_call = nat.call


def call(name, *a):
    t0 = time.perf_counter()
    _call(name, *a)
    if name == "xgs_raster_build":
        inner.append(time.perf_counter() - t0)


nat.call = call
tot = []
for i in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pr = rz._Pairs(field, pose, intr, grid.rows(), grid.cols(), rz.DEFAULT_RASTER)
    torch.cuda.synchronize()
    tot.append(time.perf_counter() - t0)
    t1 = time.perf_counter()
    pr.close()
    torch.cuda.synchronize()
    print("build ms", round(tot[-1] * 1e3, 2), "C call ms", round(inner[-1] * 1e3, 2), "close ms",
          round((time.perf_counter() - t1) * 1e3, 2))
nat.profile_enable(True)
pr = rz._Pairs(field, pose, intr, grid.rows(), grid.cols(), rz.DEFAULT_RASTER)
torch.cuda.synchronize()
print("device span of raster_build ms", nat.profile_read("raster_build"))
