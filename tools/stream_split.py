"""C4 per-frame latency split: grid_sample vs the VQ step (profiling aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200 import _native as nat

torch.cuda.set_device(0)
orig_sample = None
from paper_2603_09632_b200 import grid as G
from paper_2603_09632_b200 import distributed as DD
tg, tv = [], []
_s, _v = G.GridSampler.sample, DD.DataParallelVQ.step


def wrap(fn, acc):
    def f(*a, **k):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = fn(*a, **k)
        e1.record()
        torch.cuda.synchronize()
        acc.append(e0.elapsed_time(e1))
        return r
    return f


G.GridSampler.sample = wrap(_s, tg)
DD.DataParallelVQ.step = wrap(_v, tv)
print(bench.run_stream(torch, 200, torch.device("cuda", 0)))
print("grid p50", np.percentile(tg[5:], 50), "vq p50", np.percentile(tv[5:], 50))
nat.profile_enable(True)
G.GridSampler.sample, DD.DataParallelVQ.step = _s, _v
bench.run_stream(torch, 12, torch.device("cuda", 0))
nat.lib().xgs_profile_dump(b"gpurun_out/stream_tl.csv")
