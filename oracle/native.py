"""TEST INFRASTRUCTURE ONLY — ctypes binding of the C oracle (``oracle/oracle.c``).

Used by tests (big-shape parity subsets) and by bench.py's CPU baseline, where the
single-threaded C restatement is fanned out over row ranges with a thread pool
(ctypes releases the GIL during the call).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

DT = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
DT_BF16 = 2


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.xgs_oracle_sqdist.argtypes = [vp, i32, i64, i64, dp, i64, dp]
        L.xgs_oracle_assign.argtypes = [vp, i32, i64, i64, dp, i64, dp]
        L.xgs_oracle_accumulate.argtypes = [vp, i32, i64, i64, dp, i64, dp, dp]
        L.xgs_oracle_backproject.argtypes = [dp, dp, dp, dp, dp, dp, i64, dp]
        L.xgs_oracle_grid_keys.argtypes = [vp, i64, i64, i64, dp, dp, dp, ctypes.c_double, vp, dp]
        L.xgs_oracle_pairwise_sum.argtypes = [dp, i64]
        L.xgs_oracle_pairwise_sum.restype = ctypes.c_double
        _LIB = L
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dtype_code(x, bf16):
    if bf16:
        assert x.dtype == np.uint16
        return DT_BF16
    return DT[x.dtype]


def pairwise_sum(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().xgs_oracle_pairwise_sum(_ptr(a), a.size)


def sqdist(x, E, bf16=False):
    x = np.ascontiguousarray(x)
    E = np.ascontiguousarray(E, dtype=np.float64)
    N, D = x.shape
    out = np.empty((N, E.shape[0]))
    lib().xgs_oracle_sqdist(_ptr(x), _dtype_code(x, bf16), N, D, _ptr(E), E.shape[0], _ptr(out))
    return out


def assign(x, E, threads=1, bf16=False):
    """Reference assign_batch (vq.py:84-87) over row ranges on ``threads`` cores."""
    x = np.ascontiguousarray(x)
    if not bf16 and x.dtype not in DT:
        x = x.astype(np.float64)
    E = np.ascontiguousarray(E, dtype=np.float64)
    N, D = x.shape
    codes = np.empty(N, dtype=np.int64)
    code = _dtype_code(x, bf16)
    L = lib()

    def run(lo, hi):
        if hi > lo:
            L.xgs_oracle_assign(ctypes.c_void_p(x.ctypes.data + lo * D * x.itemsize), code,
                                hi - lo, D, _ptr(E), E.shape[0],
                                ctypes.c_void_p(codes.ctypes.data + lo * 8))

    threads = max(1, int(threads))
    if threads == 1:
        run(0, N)
    else:
        bounds = [int(b) for b in np.linspace(0, N, threads + 1)]
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: run(bounds[i], bounds[i + 1]), range(threads)))
    return codes


def accumulate(x, codes, K, bf16=False):
    """bincount + np.add.at (vq.py:97-99) as sequential fp64 chains."""
    x = np.ascontiguousarray(x)
    if not bf16 and x.dtype not in DT:
        x = x.astype(np.float64)
    codes = np.ascontiguousarray(codes, dtype=np.int64)
    N, D = x.shape
    counts = np.empty(K)
    sums = np.empty((K, D))
    lib().xgs_oracle_accumulate(_ptr(x), _dtype_code(x, bf16), N, D, _ptr(codes), K,
                                _ptr(counts), _ptr(sums))
    return counts, sums


def backproject(R, t, intr4, u, v, depth):
    R = np.ascontiguousarray(R, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    intr4 = np.ascontiguousarray(intr4, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    depth = np.ascontiguousarray(depth, dtype=np.float64)
    out = np.empty((u.size, 3))
    lib().xgs_oracle_backproject(_ptr(R), _ptr(t), _ptr(intr4), _ptr(u), _ptr(v), _ptr(depth),
                                 u.size, _ptr(out))
    return out


def grid_keys(depth, intr4, R, t, voxel, stride=1):
    depth = np.ascontiguousarray(depth, dtype=np.float32)
    H, W = depth.shape
    keys = np.empty(H * W, dtype=np.uint64)
    pts = np.empty((H * W, 3))
    lib().xgs_oracle_grid_keys(_ptr(depth), H, W, int(stride),
                               _ptr(np.ascontiguousarray(intr4, dtype=np.float64)),
                               _ptr(np.ascontiguousarray(R, dtype=np.float64)),
                               _ptr(np.ascontiguousarray(t, dtype=np.float64)),
                               float(voxel), _ptr(keys), _ptr(pts))
    return keys, pts
