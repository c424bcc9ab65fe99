"""Timeline of one C5 step (all 67,108,864 rows on one GPU): per-scope start/end
from the library profiler, and the idle gaps of the screen between row chunks."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
import paper_2603_09632_b200 as xv

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
x, E0 = bench.c5_data(torch, 0, 1, dev)
cfg = xv.VqConfig(K=bench.C5_K, lam=bench.LAM, gamma=0.5 / bench.C5_K, delta_dead=bench.DELTA, epsilon=bench.EPS,
                  reservoir_capacity=bench.CAP)
be = CudaBackend(bench.C5_K, bench.C5_D, bench.LAM, bench.EPS)
vq = DataParallelVQ((E0, torch.zeros(bench.C5_K, dtype=torch.float64, device=dev),
                     torch.zeros(bench.C5_K, bench.C5_D, dtype=torch.float64, device=dev)), cfg,
                    np.random.default_rng(42), be)
sizes = [int(x.shape[0])]
for _ in range(3):
    vq.step(x, sizes)
torch.cuda.synchronize()
nat.profile_enable(True)
vq.step(x, sizes)
torch.cuda.synchronize()
out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5_timeline.csv"
nat.lib().xgs_profile_dump(out.encode())
rows = [l.strip().split(",") for l in open(out) if l.strip() and not l.startswith("tag")]
ev = [(t, float(a), float(b)) for t, a, b in rows]
scr = sorted((a, b) for t, a, b in ev if t == "vq_screen")
gaps = [scr[i + 1][0] - scr[i][1] for i in range(len(scr) - 1)]
span = max(b for _, _, b in ev) - min(a for _, a, _ in ev)
print("step span ms", round(span, 2), "screen launches", len(scr), "screen total ms", round(sum(b - a for a, b in scr), 2))
print("gaps between screens ms: sum", round(sum(gaps), 2), "median", round(float(np.median(gaps)), 3),
      "max", round(max(gaps), 3))
first = min(a for _, a, _ in ev)
print("before first screen ms", round(scr[0][0] - first, 2), "after last screen ms",
      round(max(b for _, _, b in ev) - scr[-1][1], 2))
for tag in sorted(set(t for t, _, _ in ev)):
    sp = [(a, b) for t, a, b in ev if t == tag]
    print(f"  {tag:14s} n={len(sp):3d} busy ms {sum(b - a for a, b in sp):8.2f}")
