"""Host-time split of PerceiverStream.step on C4 frames (replay+sync vs host work)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2603_09632_b200 import stream as S

orig_replay = None
acc = {"replay+sync": [], "total": []}


class Timed(S.PerceiverStream):
    def step(self, *a):
        t0 = time.perf_counter()
        r = super().step(*a)
        acc["total"].append((time.perf_counter() - t0) * 1e3)
        return r


_rep = torch.cuda.CUDAGraph.replay


def replay(self):
    t0 = time.perf_counter()
    _rep(self)
    torch.cuda.current_stream().synchronize()
    acc["replay+sync"].append((time.perf_counter() - t0) * 1e3)


torch.cuda.CUDAGraph.replay = replay
S.PerceiverStream = Timed
bench_mod = bench
out = bench.run_stream(torch, int(sys.argv[1]) if len(sys.argv) > 1 else 200, torch.device("cuda", 0))
for k, v in acc.items():
    v = np.array(v[5:])
    print(k, "p50 %.3f ms  mean %.3f" % (np.percentile(v, 50), v.mean()))
print(out["p50_ms"], out["mean_new_per_frame"])
