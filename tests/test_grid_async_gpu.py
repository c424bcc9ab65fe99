"""XGS_GRID_ASYNC (graph-capturable grid sampling): refused before a
synchronous batch sized the library state, refused in mean mode, and once
allowed gives the synchronous outputs with the counts in dev_status."""

import ctypes
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import ctypes, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet, _grid_ws_bytes
H, W = 48, 64
d = torch.rand(1, H, W, device="cuda") * 3 + 0.5
R = torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).contiguous()
T = torch.zeros(1, 3, dtype=torch.float64, device="cuda")
cap = H * W
flat = torch.zeros(11 * cap, dtype=torch.float64, device="cuda")
st = torch.zeros(4, dtype=torch.int64, device="cuda")
hs = VoxelHashSet(1 << 16)
b = flat.data_ptr()
def call(mode):
    fr = nat.GridFrames(1, H, W, d.data_ptr(), None, R.data_ptr(), T.data_ptr(), 40.0, 40.0, 23.5, 31.5, 0.05, 1,
                        mode, 1e-3, None, 0, 0, 0, nat.GRID_ASYNC)
    res = nat.GridResult(cap, b, b + 8 * cap, b + 16 * cap, b + 40 * cap, b + 64 * cap, b + 72 * cap, None,
                         b + 80 * cap, 0, 0, 0, 0, 0, nat.F32, st.data_ptr())
    ws = nat.workspace("g", _grid_ws_bytes(cap))
    rc = nat.lib().xgs_grid_sample(ctypes.byref(fr), hs._h, ctypes.byref(res), nat.ptr(ws), ws.numel(), nat.stream_ptr())
    return rc, res
rc0, _ = call(0)            # fresh process: no library state yet
rc1, _ = call(1)            # mean mode
print("RC", rc0, rc1)
'''


def test_async_refused_without_state_and_in_mean_mode(cuda):
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RC")][0]
    rc0, rc1 = (int(v) for v in line.split()[1:])
    assert rc0 == 4 and rc1 == 4      # XGS_NOT_SUPPORTED


def test_async_matches_sync(cuda):
    import torch

    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet, _grid_ws_bytes
    rng = np.random.default_rng(3)
    H, W = 60, 80
    frames = [torch.from_numpy(rng.uniform(0.5, 4.0, (1, H, W)).astype(np.float32)).cuda() for _ in range(3)]
    R = torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).contiguous()
    Ts = [torch.tensor([[0.01 * i, 0.0, 0.0]], dtype=torch.float64, device="cuda") for i in range(3)]
    intr = (50.0, 50.0, 29.5, 39.5)
    # synchronous reference run (also sizes the library state)
    gs = GridSampler(intr, 0.04, occupied=VoxelHashSet(1 << 16))
    ref = [gs.sample(f, (R, t)).to_numpy() for f, t in zip(frames, Ts)]
    # async run on a fresh map
    hs = VoxelHashSet(1 << 16)
    cap = H * W
    flat = torch.zeros(11 * cap, dtype=torch.float64, device="cuda")
    st = torch.zeros(4, dtype=torch.int64, device="cuda")
    b = flat.data_ptr()
    for f, t, rr in zip(frames, Ts, ref):
        fr = nat.GridFrames(1, H, W, f.data_ptr(), None, R.data_ptr(), t.data_ptr(), *intr, 0.04, 1, 0, 1e-3, None, 0,
                            0, 0, nat.GRID_ASYNC)
        res = nat.GridResult(cap, b, b + 8 * cap, b + 16 * cap, b + 40 * cap, b + 64 * cap, b + 72 * cap, None,
                             b + 80 * cap, 0, 0, 0, 0, 0, nat.F32, st.data_ptr())
        ws = nat.workspace("g_async", _grid_ws_bytes(cap))
        nat.call("xgs_grid_sample", ctypes.byref(fr), hs._h, ctypes.byref(res), nat.ptr(ws), ws.numel(),
                 nat.stream_ptr())
        assert res.n_new == -1                      # counts are on the device
        torch.cuda.synchronize()
        n_new, n_valid, n_vox, err = (int(v) for v in st.cpu())
        assert err == 0 and n_new == len(rr["pid"]) and n_valid == rr["n_valid"] and n_vox == rr["n_voxels"]
        assert np.array_equal(flat[cap:cap + n_new].view(torch.int64).cpu().numpy(), rr["pid"])
        assert np.array_equal(flat[2 * cap:2 * cap + 3 * n_new].cpu().numpy().reshape(-1, 3), rr["mu"])
