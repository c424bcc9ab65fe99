"""C4 frame: GPU time of the graph replay alone vs the host step() wall clock (profiling aid)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
orig = None
import paper_2603_09632_b200.stream as S

gpu_ms, host_ms, post_ms = [], [], []
_step = S.PerceiverStream.step


def step(self, *a, **k):
    if self.graph is None:
        return _step(self, *a, **k)
    g = self.graphs[self._cur]
    R0 = g.replay
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def rep():
        e0.record()
        R0()
        e1.record()
    g.replay = rep
    t0 = time.perf_counter()
    out = _step(self, *a, **k)
    t1 = time.perf_counter()
    g.replay = R0
    torch.cuda.synchronize()
    gpu_ms.append(e0.elapsed_time(e1))
    host_ms.append((t1 - t0) * 1e3)
    return out


S.PerceiverStream.step = step
r = bench.run_stream(torch, int(sys.argv[1]) if len(sys.argv) > 1 else 300, torch.device("cuda", 0))
print("bench p50", r["p50_ms"], "p99", r["p99_ms"])
print("graph GPU ms p50", float(np.median(gpu_ms)), "p99", float(np.percentile(gpu_ms, 99)))
print("step host ms p50", float(np.median(host_ms)))
