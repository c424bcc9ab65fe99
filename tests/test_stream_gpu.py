"""The graph-captured per-frame stream (paper_2603_09632_b200/stream.py) against
the same frames through the public, synchronous path: GridSampler.sample(...,
features=...) then online_step on the returned features (vq.py:193-212) --
per-frame new-voxel counts, revived codes and the final codebook bit-identical,
including frames whose new points overflow the graph's VQ window (rolled back
and redone synchronously) and frames with no new points."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _frames(torch, n, H, W, C, Hf, Wf, seed=5):
    from paper_2603_09632_b200 import synth
    rng = np.random.default_rng(seed)
    planes = synth.random_planes(rng, 5, centre=np.array([0.0, 0.0, 2.5]), spread=2.0)
    poses = synth.random_walk_trajectory(n, rng, step_t=0.01, step_deg=1.0)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    cent = torch.randn(16, C, generator=g, device="cuda")
    cent /= cent.norm(dim=1, keepdim=True)
    intr = (0.8 * W, 0.8 * W, (H - 1) / 2, (W - 1) / 2)
    out = []
    for i, p in enumerate(poses):
        R = torch.tensor(p.rotation, device="cuda")
        t = torch.tensor(p.translation, device="cuda")
        sph = [(p.camera_center() + p.rotation.T @ np.array([rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5),
                                                              rng.uniform(1.5, 3.0)]), rng.uniform(0.1, 0.4))]
        if i % 5 == 4:   # some frames bring a large new object (overflow the small VQ window)
            sph.append((p.camera_center() + p.rotation.T @ np.array([0.0, 0.0, 2.0]), 0.9))
        d = synth.render_depth_torch(torch, R, t, intr, H, W, planes, sph).float()
        d = torch.where(torch.rand(d.shape, generator=g, device="cuda") < 0.05, torch.zeros_like(d), d)
        col = torch.randint(0, 256, (H, W, 3), generator=g, device="cuda", dtype=torch.uint8)
        f = cent[torch.randint(0, 16, (Hf * Wf,), generator=g, device="cuda")] + 0.1 * torch.randn(
            Hf * Wf, C, generator=g, device="cuda")
        f = (f / f.norm(dim=1, keepdim=True)).T.reshape(C, Hf, Wf).contiguous()
        out.append((d, (R, t), col, f))
    if len(out) > 7:   # a frame identical to the previous one: nothing new
        out[7] = out[6]
    return out, intr


def test_stream_graph_matches_sync_pipeline(cuda):
    import torch

    import paper_2603_09632_b200 as xv
    from paper_2603_09632_b200.grid import GridSampler, VoxelHashSet
    from paper_2603_09632_b200.stream import PerceiverStream
    H, W, C, Hf, Wf, K = 96, 128, 32, 12, 16, 64
    frames, intr = _frames(torch, 14, H, W, C, Hf, Wf)
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    E0 = torch.randn(K, C, generator=g, device="cuda", dtype=torch.float64)
    E0 /= E0.norm(dim=1, keepdim=True)
    cfg = xv.VqConfig(K=K, lam=0.9, gamma=0.5 / K, delta_dead=0.05, reservoir_capacity=512)

    def cb0():
        return xv.Codebook._make(E0.clone(), torch.zeros(K, dtype=torch.float64, device="cuda"),
                                 torch.zeros(K, C, dtype=torch.float64, device="cuda"), 0.9, 1e-5,
                                 xv.FeatureReservoir(512, C))

    st = PerceiverStream(intr, H, W, 0.03, cb0(), cfg, (C, Hf, Wf), np.random.default_rng(3), map_capacity=1 << 20,
                         vq_capacity=256)
    got = [st.step(*fr) for fr in frames]
    # the synchronous public path
    gs = GridSampler(intr, 0.03, occupied=VoxelHashSet(1 << 20))
    cb = cb0()
    rng = np.random.default_rng(3)
    ref_n, ref_rev = [], []
    for d, (R, t), col, f in frames:
        r = gs.sample(d, (R[None], t[None]), col, features=f)
        ref_n.append(len(r))
        if len(r):
            cb, res = xv.online_step(cb, r.feature, cfg, rng)
            ref_rev.append(res.revived)
        else:
            ref_rev.append([])
    assert [o.n_new for o in got] == ref_n
    assert [o.revived for o in got] == ref_rev
    assert any(o.graph for o in got) and any(not o.graph for o in got[1:])     # both paths exercised
    assert any(n == 0 for n in ref_n) and any(n > 256 for n in ref_n)
    assert any(len(r) for r in ref_rev)                                          # revival exercised
    mine = st.codebook()
    for a, b in ((mine.E, cb.E), (mine.N, cb.N), (mine.M, cb.M)):
        assert torch.equal(a, b)
    # the reservoir FIFO the graph appends to (xgs_vq_ring_write_dev) equals the synchronous one
    assert len(mine.reservoir) == len(cb.reservoir)
    assert np.array_equal(mine.reservoir.as_array(), cb.reservoir.as_array())
