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


def test_grid_graph_replays_match_sync_and_snapshot_restore(cuda):
    """GridGraph: batches written into the graph's buffers and replayed give
    the synchronous sampler's outputs (keys, pids, mu, colour, scale, depth,
    features) on a twin map; VoxelHashSet.copy_from restores a map snapshot,
    after which a replay reproduces the same batch exactly."""
    import torch

    from paper_2603_09632_b200 import synth
    from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet
    rng = np.random.default_rng(11)
    H, W, F = 48, 128, 2
    intr4 = (0.8 * W, 0.8 * W, (H - 1) / 2, (W - 1) / 2)
    planes = synth.random_planes(rng, 5, spread=3.0)
    poses = synth.circle_trajectory(3 * F, radius=2.0, step_deg=5.0)
    D = np.empty((3 * F, H, W), np.float32)
    C = np.empty((3 * F, H, W, 3), np.uint8)
    for i, p in enumerate(poses):
        D[i], C[i] = synth.rgbd_frame(rng, p, intr4, H, W, planes=planes, noise=0.003, zero_frac=0.05)
    R = np.stack([p.rotation for p in poses])
    T = np.stack([p.translation for p in poses])
    P = rng.normal(size=(3 * F, 6, 6, 16)).astype(np.float32)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    batch = lambda b: (dev(D[b * F:(b + 1) * F]), (dev(R[b * F:(b + 1) * F]), dev(T[b * F:(b + 1) * F])),
                       dev(C[b * F:(b + 1) * F]), dev(P[b * F:(b + 1) * F]))
    ref_gs = GridSampler(intr4, 0.03, occupied=VoxelHashSet(1 << 16))
    gr_gs = GridSampler(intr4, 0.03, occupied=VoxelHashSet(1 << 16))
    d0, p0, c0, f0 = batch(0)
    gg = GridGraph(gr_gs, d0, p0, c0, f0)
    r0 = ref_gs.sample(d0, p0, c0, features=f0).to_numpy()
    g0 = gg.first.to_numpy()
    assert np.array_equal(r0["key"], g0["key"]) and len(r0["key"]) > 0
    snap = VoxelHashSet(1 << 16)
    snap.copy_from(gr_gs.occupied)                      # map after batch 0
    outs = []
    for b in (1, 2):
        d, (Rb, Tb), c, f = batch(b)
        gg.depth.copy_(d)
        gg.R.copy_(Rb.reshape(-1, 9))
        gg.T.copy_(Tb)
        gg.color.copy_(c)
        gg.features.copy_(f)
        gg.replay()
        got = gg.result().to_numpy()
        ref = ref_gs.sample(d, (Rb, Tb), c, features=f).to_numpy()
        assert got["n_valid"] == ref["n_valid"] and got["n_voxels"] == ref["n_voxels"]
        for name in ("key", "pid", "mu", "color", "scale", "depth", "feature"):
            assert np.array_equal(got[name], ref[name]), (b, name)
        outs.append(got)
    # restore the map as it was after batch 0 and replay batch 2 as if batch 1 never happened
    gr_gs.occupied.copy_from(snap)
    gg.replay()
    again = gg.result().to_numpy()
    twin = GridSampler(intr4, 0.03, occupied=VoxelHashSet(1 << 16))
    twin.occupied.copy_from(snap)
    d, (Rb, Tb), c, f = batch(2)
    ref2 = twin.sample(d, (Rb, Tb), c, features=f).to_numpy()
    assert len(again["key"]) >= len(outs[1]["key"])
    for name in ("key", "pid", "mu", "feature"):
        assert np.array_equal(again[name], ref2[name]), name
    with pytest.raises(Exception):
        VoxelHashSet(1 << 20).copy_from(snap)            # capacities differ


def test_grid_graph_survives_state_growth(cuda):
    """A captured GridGraph keeps working after a much larger synchronous batch
    grew the library's per-device grid state (outgrown buffers are retired,
    not freed, once an async call happened)."""
    import torch

    from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet
    rng = np.random.default_rng(21)
    H, W = 48, 64
    intr = (50.0, 50.0, 23.5, 31.5)
    R = torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).contiguous()
    T = torch.zeros(1, 3, dtype=torch.float64, device="cuda")
    frame = lambda: torch.from_numpy(rng.uniform(0.5, 4.0, (1, H, W)).astype(np.float32)).cuda()
    gs = GridSampler(intr, 0.03, occupied=VoxelHashSet(1 << 16))
    twin = GridSampler(intr, 0.03, occupied=VoxelHashSet(1 << 16))
    d0 = frame()
    gg = GridGraph(gs, d0, (R, T))
    twin.sample(d0, (R, T))
    # a large synchronous batch on another map: ~1.2M distinct 1 mm voxels
    big = torch.from_numpy(rng.uniform(0.5, 5.0, (4, 480, 640)).astype(np.float32)).cuda()
    GridSampler((525.0, 525.0, 239.5, 319.5), 0.001, occupied=VoxelHashSet(1 << 22)).sample(
        big, (torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).repeat(4, 1),
              torch.zeros(4, 3, dtype=torch.float64, device="cuda")))
    for _ in range(2):
        d = frame()
        gg.depth.copy_(d)
        gg.replay()
        got = gg.result().to_numpy()
        ref = twin.sample(d, (R, T)).to_numpy()
        assert got["n_voxels"] == ref["n_voxels"] and len(got["key"]) == len(ref["key"])
        for name in ("key", "pid", "mu", "scale", "depth"):
            assert np.array_equal(got[name], ref[name]), name


def test_map_captured_by_a_graph_refuses_to_grow(cuda):
    """After an XGS_GRID_ASYNC call used a map, a call that would have to grow
    it fails loudly (a captured graph would keep using the old table)."""
    import torch

    from paper_2603_09632_b200.errors import NativeError
    from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet
    rng = np.random.default_rng(5)
    d = torch.from_numpy(rng.uniform(0.5, 4.0, (1, 48, 64)).astype(np.float32)).cuda()
    R = torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).contiguous()
    T = torch.zeros(1, 3, dtype=torch.float64, device="cuda")
    hs = VoxelHashSet(1 << 13)
    GridGraph(GridSampler((50.0, 50.0, 23.5, 31.5), 0.03, occupied=hs), d, (R, T))
    hs.insert(np.arange(1, 1000, dtype=np.uint64))            # fits: fine
    with pytest.raises(NativeError, match="cannot grow"):
        hs.insert(np.arange(1, 200_000, dtype=np.uint64))


def test_grid_graph_refuses_mean_mode(cuda):
    import torch

    from paper_2603_09632_b200.errors import InvalidInputError
    from paper_2603_09632_b200.grid import GridGraph, GridSampler, VoxelHashSet
    d = torch.full((1, 16, 32), 2.0, device="cuda")
    R = torch.eye(3, dtype=torch.float64, device="cuda").reshape(1, 9).contiguous()
    T = torch.zeros(1, 3, dtype=torch.float64, device="cuda")
    with pytest.raises(InvalidInputError):
        GridGraph(GridSampler((20.0, 20.0, 7.5, 15.5), 0.05, mode="mean", occupied=VoxelHashSet(1 << 12)), d, (R, T))
