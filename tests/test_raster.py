"""§8(f) #2 lattice rasterizer + VJP: oracle pinned to the reference's golden
vectors (CPU) and the CUDA drop-in against the same vectors (GPU).

Tolerances: pair identities (gauss, pixel, alive) and argmax ids are exact;
fp64 values differ from the reference only through libm vs CUDA ulps (exp,
log1p, atan2, cos, sin) and the reference's global cumsum of log
transmittance (the CUDA path sums per pixel), so weights / renders /
gradients are compared at rtol 1e-9.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import raster as orz

TAGS = ("dense", "bbox", "grid")


def _case(g, tag):
    H, W, s, oh, ow = (int(v) for v in g[f"{tag}_grid"])
    rows = oh + s * np.arange(max(0, 1 + (H - 1 - oh) // s))
    cols = ow + s * np.arange(max(0, 1 + (W - 1 - ow) // s))
    i = g[f"{tag}_intr"]
    return rows, cols, (i[0], i[1], i[2], i[3], i[6], i[7])


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_pinned_to_reference(tag):
    g = golden("raster")
    rows, cols, intr = _case(g, tag)
    bp = orz.blend_pairs(g[f"{tag}_mu"], g[f"{tag}_quat"], g[f"{tag}_scale"], g[f"{tag}_opacity"], g[f"{tag}_R"],
                         g[f"{tag}_t"], intr, rows, cols)
    names = ("gauss", "pixel", "weight", "alpha_prime", "t_before", "alive", "depth")
    for name, v in zip(names, bp):
        ref = g[f"{tag}_bp_{name}"]
        if name in ("gauss", "pixel", "alive"):
            assert np.array_equal(v, ref), name
        else:
            assert np.allclose(v, ref, rtol=1e-12, atol=1e-300), name
    chan = orz.accumulate(bp[0], bp[1], bp[2], g[f"{tag}_payload"], rows.size * cols.size)
    assert np.allclose(chan.reshape(g[f"{tag}_chan"].shape), g[f"{tag}_chan"], rtol=1e-12, atol=1e-14)


def _objs(g, tag):
    from paper_2603_09632_b200.core import CameraIntrinsics, CameraPose, Codebook, FeatureReservoir, GaussianField
    field = GaussianField(**{k: g[f"{tag}_{k}"] for k in ("mu", "quat", "scale", "opacity", "color", "logits")})
    i = g[f"{tag}_intr"]
    intr = CameraIntrinsics(fx=i[0], fy=i[1], cx=i[2], cy=i[3], height=int(i[4]), width=int(i[5]), near=i[6],
                            far=i[7])
    pose = CameraPose(g[f"{tag}_R"], g[f"{tag}_t"])
    E = g[f"{tag}_E"]
    cb = Codebook(E=E, N=np.zeros(E.shape[0]), M=np.zeros_like(E), lam=0.96, epsilon=1e-5,
                  reservoir=FeatureReservoir(16, E.shape[1]))
    return field, pose, intr, cb


@pytest.mark.gpu
@pytest.mark.parametrize("tag", TAGS)
def test_gpu_matches_reference_golden(cuda, tag):
    from paper_2603_09632_b200 import rasterizer as rz
    from paper_2603_09632_b200.supervision import GridSpec
    g = golden("raster")
    field, pose, intr, cb = _objs(g, tag)
    H, W, s, oh, ow = (int(v) for v in g[f"{tag}_grid"])
    grid = GridSpec(H=H, W=W, s=s, o_h=oh, o_w=ow)
    bp = rz.build_blend_pairs(field, pose, intr, grid.rows(), grid.cols())
    for name in ("gauss", "pixel", "alive"):
        assert np.array_equal(getattr(bp, name), g[f"{tag}_bp_{name}"]), name
    for name in ("weight", "alpha_prime", "t_before", "depth"):
        assert np.allclose(getattr(bp, name), g[f"{tag}_bp_{name}"], rtol=1e-9, atol=1e-300), name
    assert bp.blend_steps == int(g[f"{tag}_bp_steps"])
    if s == 1:
        r = rz.render(field, pose, intr)
        for name in ("color", "depth", "alpha"):
            assert np.allclose(getattr(r, name), g[f"{tag}_r_{name}"], rtol=1e-9, atol=1e-12), name
        assert r.blend_steps == int(g[f"{tag}_steps"])
        assert np.array_equal(rz.render_argmax_ids(field, pose, intr), g[f"{tag}_argmax"])
    chan = rz.render_channels_grid(field, g[f"{tag}_payload"], pose, intr, grid)
    assert np.allclose(chan.data, g[f"{tag}_chan"], rtol=1e-9, atol=1e-12)
    feat = rz.render_features_grid(field, cb, pose, intr, grid)
    assert np.allclose(feat.data, g[f"{tag}_feat"], rtol=1e-9, atol=1e-12)
    fgr = rz.feature_gradients(field, cb, pose, intr, grid, g[f"{tag}_up"])
    assert np.allclose(fgr.feature_grads, g[f"{tag}_fg"], rtol=1e-9, atol=1e-12)
    assert np.allclose(fgr.logit_grads, g[f"{tag}_lg"], rtol=1e-9, atol=1e-12)


@pytest.mark.gpu
def test_gpu_edge_cases(cuda):
    from paper_2603_09632_b200 import rasterizer as rz
    from paper_2603_09632_b200.core import CameraIntrinsics, CameraPose, GaussianField
    from paper_2603_09632_b200.errors import EmptySceneError, InvalidInputError
    from paper_2603_09632_b200.supervision import GridSpec
    intr = CameraIntrinsics(fx=20.0, fy=20.0, cx=7.5, cy=9.5, height=16, width=20)
    pose = CameraPose.identity()
    empty = GaussianField(mu=np.zeros((0, 3)), quat=np.zeros((0, 4)), scale=np.zeros((0, 3)), opacity=np.zeros(0),
                          color=np.zeros((0, 3)), logits=np.zeros((0, 3)))
    with pytest.raises(EmptySceneError):
        rz.render(empty, pose, intr)
    bp = rz.build_blend_pairs(empty, pose, intr, np.arange(4), np.arange(4))
    assert bp.gauss.size == 0 and bp.n_pixels == 16
    # single opaque Gaussian on axis (test_rasterizer.py:27-34): alpha ~ opacity at the centre
    one = GaussianField(mu=[[0.0, 0.0, 2.0]], quat=[[1.0, 0, 0, 0]], scale=[[0.2, 0.2, 0.2]], opacity=[0.9],
                        color=[[1.0, 0.5, 0.25]], logits=np.zeros((1, 3)))
    r = rz.render(one, pose, intr)
    assert 0.5 < r.alpha[7, 9] <= 0.9 and r.alpha.max() <= 0.9 + 1e-12 and np.all(r.alpha >= 0)
    assert np.allclose(r.color[:, 7, 9], r.alpha[7, 9] * np.array([1.0, 0.5, 0.25]), rtol=1e-12)
    assert np.allclose(r.depth[7, 9], r.alpha[7, 9] * 2.0, rtol=1e-12)
    # behind the camera -> no pairs, argmax -1 everywhere
    behind = GaussianField(mu=[[0.0, 0.0, -1.0]], quat=[[1.0, 0, 0, 0]], scale=[[0.2, 0.2, 0.2]], opacity=[0.9],
                           color=[[1.0, 0.5, 0.25]], logits=np.zeros((1, 3)))
    assert np.all(rz.render_argmax_ids(behind, pose, intr) == -1)
    # empty lattice -> empty map; shape mismatch raises
    m = rz.render_channels_grid(one, np.ones((1, 2)), pose, intr, GridSpec(H=0, W=5))
    assert m.data.shape == (2, 0, 5)
    with pytest.raises(InvalidInputError):
        rz.render_channels_grid(one, np.ones((2, 2)), pose, intr, GridSpec(H=16, W=20))


@pytest.mark.gpu
def test_gpu_large_scene_matches_oracle(cuda):
    """20k Gaussians on a 120x160 frame, stride-2 lattice: pairs and channels vs the oracle."""
    from paper_2603_09632_b200 import rasterizer as rz
    from paper_2603_09632_b200.core import CameraIntrinsics, CameraPose, GaussianField
    rng = np.random.default_rng(11)
    n, H, W = 20000, 120, 160
    mu = np.column_stack([rng.uniform(-2, 2, n), rng.uniform(-2, 2, n), rng.uniform(0.2, 6, n)])
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scale = np.exp(rng.uniform(np.log(0.005), np.log(0.1), (n, 3)))
    op = rng.uniform(0.1, 1.0, n)
    field = GaussianField(mu=mu, quat=q, scale=scale, opacity=op, color=rng.random((n, 3)), logits=np.zeros((n, 2)))
    intr = CameraIntrinsics(fx=150.0, fy=150.0, cx=59.5, cy=79.5, height=H, width=W)
    pose = CameraPose.identity()
    rows, cols = np.arange(1, H, 2), np.arange(0, W, 2)
    bp = rz.build_blend_pairs(field, pose, intr, rows, cols)
    ref = orz.blend_pairs(mu, q, scale, op, np.eye(3), np.zeros(3), (150.0, 150.0, 59.5, 79.5, 0.05, 100.0), rows,
                          cols)
    assert np.array_equal(bp.gauss, ref[0]) and np.array_equal(bp.pixel, ref[1])
    assert np.allclose(bp.weight, ref[2], rtol=1e-9, atol=1e-300)
