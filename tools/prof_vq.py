"""Profiling driver: a few online_steps at the C2 shape (for ncu runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
import paper_2603_09632_b200 as xv

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
torch.cuda.set_device(0)
x, E0 = bench.make_data(torch, 0, torch.device("cuda", 0))
K, D = bench.K, bench.D
cfg = xv.VqConfig(K=K, lam=bench.LAM, gamma=0.5 / K, delta_dead=bench.DELTA, reservoir_capacity=bench.CAP)
vq = DataParallelVQ((E0, torch.zeros(K, dtype=torch.float64, device="cuda"),
                     torch.zeros(K, D, dtype=torch.float64, device="cuda")), cfg, np.random.default_rng(12),
                    CudaBackend(K, D, bench.LAM, bench.EPS))
for _ in range(steps):
    vq.step(x, [x.shape[0]])
torch.cuda.synchronize()
print("done")
