"""Host-side cost of one DataParallelVQ.step at C2 (no GPU sync except the
revival read-back): wall time per step vs the device time per step."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
import paper_2603_09632_b200 as xv

torch.cuda.set_device(0)
x, E0 = bench.make_data(torch, 0, torch.device("cuda", 0))
K, D = bench.K, bench.D
cfg = xv.VqConfig(K=K, lam=bench.LAM, gamma=0.5 / K, delta_dead=bench.DELTA, reservoir_capacity=bench.CAP)
vq = DataParallelVQ((E0, torch.zeros(K, dtype=torch.float64, device="cuda"),
                     torch.zeros(K, D, dtype=torch.float64, device="cuda")), cfg, np.random.default_rng(12),
                    CudaBackend(K, D, bench.LAM, bench.EPS))
for _ in range(25):
    vq.step(x, [x.shape[0]])
torch.cuda.synchronize()
import cProfile, pstats
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(20):
    vq.step(x, [x.shape[0]])
pr.disable()
torch.cuda.synchronize()
print("ms/step wall", (time.perf_counter() - t0) / 20 * 1e3)
pstats.Stats(pr).sort_stats("tottime").print_stats(14)

# GPU-idle host window: from the end of a step's read-back (the only sync) to
# the first libxgs call of the next step
from paper_2603_09632_b200 import _native as nat
be = vq.be
marks = {"sync_end": None, "gaps": [], "calls": 0}
orig_counts, orig_call = be.counts_host, nat.call


def counts_host(state):
    out = orig_counts(state)
    marks["sync_end"] = time.perf_counter()
    return out


def call(name, *args):
    if marks["sync_end"] is not None:
        marks["gaps"].append((time.perf_counter() - marks["sync_end"]) * 1e6)
        marks["sync_end"] = None
    return orig_call(name, *args)


be.counts_host = counts_host
nat.call = call
import paper_2603_09632_b200.vq as xvq
xvq.nat.call = call
for _ in range(50):
    vq.step(x, [x.shape[0]])
torch.cuda.synchronize()
g = np.array(marks["gaps"][1:])
print("host window us: p50 %.1f mean %.1f max %.1f (n=%d)" % (np.median(g), g.mean(), g.max(), g.size))
