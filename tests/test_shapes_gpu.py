"""Parity at the BASELINE shapes (not just small frames / small codebooks).

* C3: 4 frames of 1280x720 with the bench's 1050 px intrinsics, voxel 0.01
  and 0.05 m, against a scene-derived ~4M-voxel running map (bench.grid_warm_map:
  the same scene sampled from the rest of the trajectory + filler keys):
  keys, pixel ids, mu, colour, scale, depth bit-exact vs oracle/grid.py.
* C5: 20,480 bf16 rows at D=1152, K=4096 (4096-centre mixture), 5 online
  steps, against the C restatement (oracle.c, bf16=True) + the oracle's
  EMA / revival: E, N, M bit-exact after every step, then the codes.
* C2: 20 online steps on a 65,536-row subset of the C2 distribution (D=512
  fp32, K=1024) bit-exact against the oracle.
"""

import os
import sys

import numpy as np
import pytest

from oracle import grid as og
from oracle import native as on
from oracle import vq as ov

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
THREADS = os.cpu_count() or 4


@pytest.fixture(scope="module")
def c3_frames():
    import bench
    return bench.grid_scene(frames=4)


@pytest.mark.parametrize("voxel", [0.01, 0.05])
def test_c3_shape_against_scene_map(cuda, c3_frames, voxel):
    import torch

    import bench
    from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet
    D, C, R, T = c3_frames
    warm, n_scene, _ = bench.grid_warm_map(torch, voxel, max_frames=120)
    hs = VoxelHashSet(bench.GRID_MAP + D.size)
    hs.insert(warm)
    got = GridSampler(bench.GRID_INTR, voxel, occupied=hs).sample(torch.from_numpy(D).cuda(),
                                                                  (torch.from_numpy(R).cuda(),
                                                                   torch.from_numpy(T).cuda()),
                                                                  torch.from_numpy(C).cuda()).to_numpy()
    occ = set(int(k) for k in warm.cpu().numpy().view(np.uint64))
    ref = og.grid_sample([(D[f], C[f], R[f], T[f]) for f in range(D.shape[0])], np.array(bench.GRID_INTR), voxel,
                         occ)
    assert got["n_valid"] == ref["n_valid"] and got["n_voxels"] == ref["n_voxels"]
    assert 0 < len(got["key"]) < got["n_voxels"]          # the scene map rejects part of the batch
    for name in ("key", "pid", "mu", "color", "scale", "depth"):
        assert np.array_equal(got[name], ref[name]), name
    hs.close()


def _mixture_bf16(torch, n, d, centres, sigma, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    Cm = torch.randn(centres, d, generator=g, device="cuda")
    Cm /= Cm.norm(dim=1, keepdim=True)
    x = Cm[torch.randint(0, centres, (n,), generator=g, device="cuda")] + sigma * torch.randn(
        n, d, generator=g, device="cuda")
    return (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16), Cm


def _oracle_step(oc, xb_host, K, bf16, rng):
    oc.reservoir.extend(xb_host if not bf16 else _bf16_to_f64(xb_host))
    codes = on.assign(xb_host, oc.E, threads=THREADS, bf16=bf16)
    counts, sums = on.accumulate(xb_host, codes, K, bf16=bf16)
    oc = ov.ema_step(oc, counts, sums)
    oc, rev, _ = ov.revive_dead_codes(oc, 1e-3, rng)
    return oc, rev


def _bf16_to_f64(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def test_c5_shape_bf16_k4096(cuda):
    import torch

    import paper_2603_09632_b200 as xv
    n, d, K = 20480, 1152, 4096
    x, Cm = _mixture_bf16(torch, n, d, 4096, 0.05, 40)
    g = torch.Generator(device="cuda")
    g.manual_seed(41)
    e = Cm[torch.randint(0, 4096, (K,), generator=g, device="cuda")] + 0.05 * torch.randn(K, d, generator=g,
                                                                                        device="cuda")
    E0 = (e / e.norm(dim=1, keepdim=True)).to(torch.bfloat16).double()
    cfg = xv.VqConfig(K=K, lam=0.99, gamma=0.5 / K, delta_dead=1e-3)
    cb = xv.Codebook._make(E0.clone(), torch.zeros(K, dtype=torch.float64, device="cuda"),
                           torch.zeros(K, d, dtype=torch.float64, device="cuda"), 0.99, 1e-5,
                           xv.FeatureReservoir(4096, d))
    xh = x.view(torch.int16).cpu().numpy().view(np.uint16)
    oc = ov.OracleCodebook(E0.cpu().numpy(), np.zeros(K), np.zeros((K, d)), 0.99, 1e-5, ov.OracleReservoir(4096, d))
    r1, r2 = np.random.default_rng(4), np.random.default_rng(4)
    for step in range(5):
        cb, res = xv.online_step(cb, x, cfg, r1)
        oc, rev = _oracle_step(oc, xh, K, True, r2)
        c = cb.to_numpy()
        assert np.array_equal(c.N, oc.N) and np.array_equal(c.M, oc.M) and np.array_equal(c.E, oc.E), step
        assert res.revived == rev
    codes = xv.assign_batch(x, cb).cpu().numpy()
    assert np.array_equal(codes, on.assign(xh, oc.E, threads=THREADS, bf16=True))


def test_c2_shape_20_steps(cuda):
    import torch

    import bench
    import paper_2603_09632_b200 as xv
    x, E0 = bench.make_data(torch, 0, torch.device("cuda", 0))
    n = 65536
    xs = x[:n].contiguous()
    del x
    K, d = bench.K, bench.D
    cfg = xv.VqConfig(K=K, lam=0.99, gamma=0.5 / K, delta_dead=1e-3)
    cb = xv.Codebook._make(E0.clone(), torch.zeros(K, dtype=torch.float64, device="cuda"),
                           torch.zeros(K, d, dtype=torch.float64, device="cuda"), 0.99, 1e-5,
                           xv.FeatureReservoir(4096, d))
    xh = xs.cpu().numpy()
    oc = ov.OracleCodebook(E0.cpu().numpy(), np.zeros(K), np.zeros((K, d)), 0.99, 1e-5, ov.OracleReservoir(4096, d))
    r1, r2 = np.random.default_rng(12), np.random.default_rng(12)
    revived = 0
    for step in range(20):
        cb, res = xv.online_step(cb, xs, cfg, r1)
        oc, rev = _oracle_step(oc, xh, K, False, r2)
        assert res.revived == rev, step
        revived += len(rev)
    c = cb.to_numpy()
    assert np.array_equal(c.N, oc.N) and np.array_equal(c.M, oc.M) and np.array_equal(c.E, oc.E)
    assert np.array_equal(cb.reservoir.as_array(), oc.reservoir.buf)
