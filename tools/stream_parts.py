"""C4 graph body split: each part captured in its own CUDA graph and replayed
(after the stream has run some frames), CUDA events around each replay."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200 import _native as nat
import paper_2603_09632_b200.stream as S

holder = {}
_init = S.PerceiverStream.__init__


def init(self, *a, **k):
    _init(self, *a, **k)
    holder["st"] = self


S.PerceiverStream.__init__ = init
bench.run_stream(torch, int(sys.argv[1]) if len(sys.argv) > 1 else 200, torch.device("cuda", 0))
st = holder["st"]
L = nat.lib()


def grid_part():
    nat.check(L.xgs_grid_sample(ctypes.byref(st._frames), st.occupied._h, ctypes.byref(st._result),
                                nat.ptr(st.ws_grid), st.ws_grid.numel(), nat.stream_ptr()))


def assign():
    nat.check(L.xgs_prefix_mask(nat.ptr(st.dev_status), st.vcap, nat.ptr(st.mask), nat.stream_ptr()))
    nat.check(L.xgs_vq_assign(nat.ptr(st.ofeat), nat.F32, st.vcap, st.C, st.C, nat.ptr(st.E), st.K,
                              nat.ptr(st.codes), nat.ptr(st.ws_assign), st.ws_assign.numel(), None, nat.stream_ptr()))


def accumulate():
    sums = st.packed[:st.K * st.D]
    counts = st.packed[st.K * st.D:]
    nat.check(L.xgs_vq_accumulate(nat.ptr(st.ofeat), nat.F32, st.vcap, st.C, st.C, nat.ptr(st.codes),
                                  nat.ptr(st.mask), st.K, nat.ptr(counts), nat.ptr(sums),
                                  nat.ptr(st.ws_acc), st.ws_acc.numel(), nat.stream_ptr()))


def ema_ring():
    sums = st.packed[:st.K * st.D]
    counts = st.packed[st.K * st.D:]
    Eo, No, Mo = st._S[1 - st._cur]
    nat.check(L.xgs_vq_ema(st.lam, st.eps, st.K, st.D, nat.ptr(st.N), nat.ptr(st.M), nat.ptr(counts),
                           nat.ptr(sums), nat.ptr(No), nat.ptr(Mo), nat.ptr(Eo), nat.stream_ptr()))


for name, fn in (("grid", grid_part), ("prefix+assign", assign), ("accumulate", accumulate),
                 ("ema", ema_ring), ("whole step graph", None)):
    if fn is None:
        g = st.graphs[st._cur]
    else:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.current_stream().wait_stream(s)
    ts = []
    for _ in range(30):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{name:18s} median {np.median(ts[5:]):7.1f} us")
