"""C4 step(): where the host time goes (replay call / sync wait / post-processing), profiling aid."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_09632_b200.stream as S

marks = []
_step = S.PerceiverStream.step


def step(self, *a, **k):
    if self.graph is None:
        return _step(self, *a, **k)
    g = self.graphs[self._cur]
    t = {}
    R0 = g.replay
    stream = torch.cuda.current_stream()
    S0 = stream.synchronize

    def rep():
        t["r0"] = time.perf_counter()
        R0()
        t["r1"] = time.perf_counter()

    def sync():
        t["s0"] = time.perf_counter()
        S0()
        t["s1"] = time.perf_counter()
    g.replay = rep
    stream.synchronize = sync
    torch.cuda.current_stream = lambda *a_: stream
    t0 = time.perf_counter()
    out = _step(self, *a, **k)
    t1 = time.perf_counter()
    g.replay = R0
    if "s1" in t:
        marks.append((t["r0"] - t0, t["r1"] - t["r0"], t["s0"] - t["r1"], t["s1"] - t["s0"], t1 - t["s1"]))
    return out


S.PerceiverStream.step = step
bench.run_stream(torch, int(sys.argv[1]) if len(sys.argv) > 1 else 300, torch.device("cuda", 0))
m = np.array(marks) * 1e6
print("us: pre, replay call, between, sync wait, post (median):", np.median(m, axis=0).round(1))
