"""GPU parity of the grid-sampling path: back-projection against the reference's
golden vectors, densify_and_prune against the reference on an empty map, and
the voxel sampler (keys, radix sort, first-pick / mean, occupancy, emission
order) against the CPU oracle (oracle/grid.py).  Keys, pixel ids, positions
and colours are compared bit-exactly."""

import numpy as np
import pytest

from conftest import golden
from oracle import grid as og

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def xs(cuda):
    from paper_2603_09632_b200 import grid, slam, synth
    return grid, slam, synth


def test_backproject_golden(xs):
    grid, slam, _ = xs
    from paper_2603_09632_b200.core import CameraPose
    g = golden("backproject")
    for k in range(g["R"].shape[0]):
        sel = g["pose_id"] == k
        p = slam.backproject_pixels(CameraPose(g["R"][k], g["t"][k]), g["intr"], g["u"][sel].astype(float),
                                    g["v"][sel].astype(float), g["d"][sel].astype(float))
        assert np.array_equal(p, g["p"][sel]), k
    i = int(np.nonzero(g["pose_id"] == 0)[0][0])
    one = slam.backproject(CameraPose(g["R"][0], g["t"][0]), g["intr"], float(g["u"][i]), float(g["v"][i]),
                           float(g["d"][i]))
    assert np.array_equal(one, g["p"][i])


def test_densify_empty_map_golden(xs):
    _, slam, _ = xs
    from paper_2603_09632_b200.core import CameraPose, GaussianField
    g = golden("densify")
    pose = CameraPose(g["R"], g["t"])
    win = slam.KeyframeWindow(4)
    win.insert(slam.CameraFrame(0, pose, g["color"], g["depth"]), pose)
    empty = GaussianField(mu=np.zeros((0, 3)), quat=np.zeros((0, 4)), scale=np.zeros((0, 3)), opacity=np.zeros(0),
                          color=np.zeros((0, 3)), logits=np.zeros((0, 5)))
    out = slam.densify_and_prune(empty, win, slam.SlamConfig(), K=5)
    for name, ref in (("mu", g["mu"]), ("scale", g["scale"]), ("color", g["col"]), ("opacity", g["opacity"]),
                      ("quat", g["quat"])):
        assert np.array_equal(getattr(out, name), ref), name
    assert out.generation == int(g["generation"])


def test_densify_nonempty_map_golden(xs):
    """Render-coverage skipping on a non-empty map (slam.py:608-626) through the
    GPU rasterizer: same inserted splats, prune set and order as the reference."""
    from paper_2603_09632_b200.core import CameraPose, GaussianField
    _, slam, _ = xs
    g = golden("densify")
    field = GaussianField(mu=g["f1_mu"], quat=g["f1_quat"], scale=g["f1_scale"], opacity=g["f1_opacity"],
                          color=g["f1_color"], logits=g["f1_logits"], generation=int(g["generation"]))
    pose2 = CameraPose(g["R2"], g["t2"])
    win = slam.KeyframeWindow(4)
    win.insert(slam.CameraFrame(1, pose2, g["color2"], g["depth2"]), pose2)
    out = slam.densify_and_prune(field, win, slam.SlamConfig(), K=5)
    assert len(out) == g["m2_mu"].shape[0]
    for name, ref in (("mu", g["m2_mu"]), ("scale", g["m2_scale"]), ("color", g["m2_color"]),
                      ("opacity", g["m2_opacity"])):
        assert np.array_equal(getattr(out, name), ref), name
    assert out.generation == int(g["m2_generation"])


def _scene(synth, seed, H, W, F, spheres=False):
    rng = np.random.default_rng(seed)
    intr4 = (0.8 * W, 0.8 * W, (H - 1) / 2, (W - 1) / 2)
    planes = synth.random_planes(rng, 6, spread=3.0)
    sph = [(rng.uniform(-1, 1, 3), rng.uniform(0.2, 0.6)) for _ in range(3)] if spheres else ()
    poses = synth.circle_trajectory(F, radius=2.0, step_deg=5.0)
    frames = []
    for p in poses:
        d, c = synth.rgbd_frame(rng, p, intr4, H, W, planes=planes, spheres=sph, noise=0.003, zero_frac=0.05)
        frames.append((d, c, p.rotation, p.translation))
    return frames, intr4


@pytest.mark.parametrize("mode", ["first", "mean"])
@pytest.mark.parametrize("voxel", [0.01, 0.05])
def test_grid_sample_matches_oracle(xs, mode, voxel):
    grid, _, synth = xs
    frames, intr4 = _scene(synth, 3, 96, 128, 3, spheres=True)
    gs = grid.GridSampler(intr4, voxel, mode=mode)
    D = np.stack([f[0] for f in frames])
    C = np.stack([f[1] for f in frames])
    R = np.stack([f[2] for f in frames])
    T = np.stack([f[3] for f in frames])
    got = gs.sample(D, (R, T), C).to_numpy()
    ref = og.grid_sample(frames, np.array(intr4), voxel, set(), mode=mode)
    assert got["n_valid"] == ref["n_valid"] and got["n_voxels"] == ref["n_voxels"]
    for name in ("key", "pid", "mu", "color", "scale", "depth"):
        assert np.array_equal(got[name], ref[name]), name
    if mode == "mean":
        assert np.array_equal(got["count"], ref["count"])


def _sample_both(grid, gs_args, batch, warm=None):
    """The same batch through the hash first-pick path (default) and the radix
    sort + select path (XGS_GRID_SORT=1), each on its own copy of the map."""
    import os
    out = []
    for force in ("0", "1"):
        os.environ["XGS_GRID_SORT"] = force
        try:
            gs = grid.GridSampler(*gs_args)
            if warm is not None:
                gs.occupied.insert(warm)
            r = gs.sample(*batch)
            out.append((r.to_numpy(), len(gs.occupied)))
        finally:
            os.environ.pop("XGS_GRID_SORT", None)
    return out


@pytest.mark.parametrize("W,voxel", [(128, 0.01), (128, 0.05), (130, 0.02)])
def test_grid_hash_and_sort_paths_agree(xs, W, voxel):
    """First-pick mode: the hash dedup (per-voxel atomicMin of the pixel id) and
    the sort path give identical outputs, on the fused front end (W % 4 == 0)
    and the two-kernel one (W = 130), with a pre-populated map."""
    grid, _, synth = xs
    frames, intr4 = _scene(synth, 5, 96, W, 11, spheres=True)
    batch = (np.stack([f[0] for f in frames]), (np.stack([f[2] for f in frames]), np.stack([f[3] for f in frames])),
             np.stack([f[1] for f in frames]))
    ref = og.grid_sample(frames[:1], np.array(intr4), voxel, set())
    (h, nh), (srt, ns) = _sample_both(grid, (intr4, voxel), batch, warm=ref["key"][::3])
    assert nh == ns and h["n_voxels"] == srt["n_voxels"] and h["n_valid"] == srt["n_valid"]
    for name in ("key", "pid", "mu", "color", "scale", "depth", "count"):
        assert np.array_equal(h[name], srt[name]), name
    assert h["sort_passes"] == 0 and srt["sort_passes"] > 0


@pytest.mark.parametrize("map_capacity", [1 << 20, 1 << 24])
def test_grid_hash_table_overflow_retry(xs, map_capacity):
    """A batch with far more distinct voxels than the table sized from the
    previous batch: the bounded probes overflow, pass 2 is skipped (map
    untouched) and the batch is redone on a table sized for every item.  With
    the large map the batch also skips the front-end read-back (item count
    first known at the final read-back)."""
    grid, _, _ = xs
    import torch
    rng = np.random.default_rng(5)
    intr4 = (525.0, 525.0, 239.5, 319.5)
    gs = grid.GridSampler(intr4, 0.05)
    small = np.full((1, 480, 640), 2.0, np.float32)
    gs.sample(small, (np.eye(3)[None], np.zeros((1, 3))))           # few voxels: next table is the 1M minimum
    D = rng.uniform(0.5, 5.0, (12, 480, 640)).astype(np.float32)     # ~3.7M distinct 1 mm voxels
    R = np.repeat(np.eye(3)[None], 12, 0)
    T = np.zeros((12, 3))
    gs.sample(small, (np.eye(3)[None], np.zeros((1, 3))))           # reset the table size after any earlier run
    (h, nh), (srt, ns) = _sample_both(grid, (intr4, 0.001, 1, "first", 1e-3, None, map_capacity), (D, (R, T)))
    assert h["n_voxels"] > 2_000_000 and h["n_valid"] == srt["n_valid"] and h["n_sorted"] == srt["n_sorted"]
    assert nh == ns and h["n_voxels"] == srt["n_voxels"]
    for name in ("key", "pid", "mu", "scale", "depth"):
        assert np.array_equal(h[name], srt[name]), name
    torch.cuda.synchronize()


@pytest.mark.parametrize("W,mode,with_color", [(128, "first", True), (128, "first", False), (130, "first", True),
                                                (128, "mean", True)])
def test_grid_pinned_host_frames_match_device(xs, W, mode, with_color):
    """Pinned host frames (xgs_grid_sample_h2d: frame-chunked copies inside the
    call overlapping the front end) give the same result as device frames."""
    import torch
    grid, _, synth = xs
    frames, intr4 = _scene(synth, 9, 64, W, 11, spheres=True)
    D = torch.from_numpy(np.stack([f[0] for f in frames]))
    C = torch.from_numpy(np.stack([f[1] for f in frames]))
    R = np.stack([f[2] for f in frames])
    T = np.stack([f[3] for f in frames])
    outs = []
    for pinned in (False, True):
        gs = grid.GridSampler(intr4, 0.02, mode=mode)
        d = D.pin_memory() if pinned else D.cuda()
        c = (C.pin_memory() if pinned else C.cuda()) if with_color else None
        outs.append(gs.sample(d, (R, T), c).to_numpy())
    for name in ("key", "pid", "mu", "color", "scale", "depth", "count"):
        assert np.array_equal(outs[0][name], outs[1][name]), name
    assert outs[0]["n_valid"] == outs[1]["n_valid"] and len(outs[0]["pid"]) > 0


def test_grid_incremental_and_batching(xs):
    grid, _, synth = xs
    frames, intr4 = _scene(synth, 4, 64, 80, 4)
    occ = set()
    refs = [og.grid_sample([f], np.array(intr4), 0.02, occ) for f in frames]
    # (a) frame by frame against a persistent device map
    gs = grid.GridSampler(intr4, 0.02)
    for f, ref in zip(frames, refs):
        got = gs.sample(f[0], ([f[2]], [f[3]]), f[1]).to_numpy()
        assert np.array_equal(got["key"], ref["key"]) and np.array_equal(got["mu"], ref["mu"])
    assert len(gs.occupied) == len(occ)
    # (b) the whole batch at once == sequential submission
    gs2 = grid.GridSampler(intr4, 0.02)
    got = gs2.sample(np.stack([f[0] for f in frames]), (np.stack([f[2] for f in frames]),
                                                          np.stack([f[3] for f in frames])),
                     np.stack([f[1] for f in frames])).to_numpy()
    HW = frames[0][0].size
    seq_pid = np.concatenate([r["pid"] + i * HW for i, r in enumerate(refs)])
    assert np.array_equal(got["pid"], seq_pid)
    assert np.array_equal(got["key"], np.concatenate([r["key"] for r in refs]))
    # (c) re-submitting the same frames adds nothing
    again = gs2.sample(frames[0][0], ([frames[0][2]], [frames[0][3]]), frames[0][1])
    assert len(again) == 0


def test_grid_config1_frame_and_stride(xs):
    grid, _, synth = xs
    d, c, pose, intr4 = synth.config1_frame(0)
    for stride in (1, 4):
        gs = grid.GridSampler(intr4, 0.02, stride=stride)
        got = gs.sample(d, [pose], c).to_numpy()
        ref = og.grid_sample([(d, c, pose.rotation, pose.translation)], np.array(intr4), 0.02, set(),
                             stride=stride)
        assert np.array_equal(got["pid"], ref["pid"]) and np.array_equal(got["mu"], ref["mu"])
        assert np.array_equal(got["scale"], ref["scale"])


def test_grid_edge_cases(xs):
    grid, _, _ = xs
    gs = grid.GridSampler((10.0, 10.0, 1.5, 1.5), 0.1)
    empty = gs.sample(np.zeros((4, 4), np.float32), (np.eye(3)[None], np.zeros((1, 3))))
    assert len(empty) == 0 and empty.n_valid == 0
    # NaN / negative depth are invalid (depth > 0 rule, slam.py:626)
    d = np.full((4, 4), np.nan, np.float32)
    d[0, 0] = -1.0
    d[1, 1] = 2.0
    r = gs.sample(d, (np.eye(3)[None], np.zeros((1, 3)))).to_numpy()
    assert r["pid"].tolist() == [5]
    # first pick across a voxel: all pixels at the same point -> lowest pid
    gs2 = grid.GridSampler((1e6, 1e6, 0.0, 0.0), 1.0)
    r = gs2.sample(np.full((3, 5), 1.5, np.float32), (np.eye(3)[None], np.zeros((1, 3)))).to_numpy()
    assert r["pid"].tolist() == [0] and r["n_voxels"] == 1


def test_voxel_boundaries_bit_exact(xs):
    """Depths exactly on / one float32 ulp around voxel boundaries (the floor
    fast path's guard band must fall back to the exact quotient)."""
    grid, _, _ = xs
    base = np.array([0.25 * k for k in range(1, 40)] + [0.1 * k for k in range(1, 40)], np.float32)
    d = np.concatenate([base, np.nextafter(base, np.float32(0)), np.nextafter(base, np.float32(10))])
    for H, W in ((6, d.size // 6), (6, 36)):   # 39 columns: unfused path; 36: fused fp32-filter front end
        _boundaries_case(grid, d[:H * W].reshape(H, W), H, W)


def _boundaries_case(grid, depth, H, W):
    for vs in (0.25, 0.1, 0.05, 1.0 / 3.0):
        intr = (7.0, 11.0, 2.5, 3.0)
        gs = grid.GridSampler(intr, vs)
        got = gs.sample(depth, (np.eye(3)[None], np.zeros((1, 3)))).to_numpy()
        ref = og.grid_sample([(depth, np.zeros((H, W, 3), np.uint8), np.eye(3), np.zeros(3))], np.array(intr), vs,
                             set())
        assert np.array_equal(got["key"], ref["key"]) and np.array_equal(got["pid"], ref["pid"]), vs


def test_fused_front_end_posed_boundaries(xs):
    """Fused front end (W % 4 == 0) under non-identity poses: depths chosen so
    many points land within float32 rounding of a voxel face; keys and pixel
    ids must equal the fp64 oracle bit for bit."""
    grid, _, _ = xs
    rng = np.random.default_rng(77)
    H, W, F = 24, 64, 3
    intr = (50.0, 47.0, 11.5, 31.5)
    R = []
    for _ in range(F):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        R.append(q * np.sign(np.linalg.det(q)))
    R = np.stack(R)
    T = rng.normal(scale=0.7, size=(F, 3))
    vs = 0.02
    D = np.empty((F, H, W), np.float32)
    for f in range(F):
        for u in range(H):
            for v in range(W):
                # choose depth so that the world z-coordinate sits on a voxel face
                a = np.array([(u - intr[2]) / intr[0], (v - intr[3]) / intr[1], 1.0])
                r = R[f].T @ a
                z0 = (R[f].T @ (-T[f]))[2]
                k = np.round((z0 + 1.5 * r[2]) / vs)
                dd = (k * vs - z0) / r[2] if abs(r[2]) > 1e-3 else 1.5
                D[f, u, v] = np.float32(dd if 0.2 < dd < 8 else 1.5)
    D = np.where(rng.random(D.shape) < 0.3, np.nextafter(D, np.float32(10)), D).astype(np.float32)
    frames = [(D[f], np.zeros((H, W, 3), np.uint8), R[f], T[f]) for f in range(F)]
    ref = og.grid_sample(frames, np.array(intr), vs, set())
    got = grid.GridSampler(intr, vs).sample(D, (R, T)).to_numpy()
    assert got["n_valid"] == ref["n_valid"] and got["n_voxels"] == ref["n_voxels"]
    for name in ("key", "pid", "mu"):
        assert np.array_equal(got[name], ref[name]), name


def test_radix_sort_matches_stable_argsort(xs, cuda):
    import torch
    grid, _, _ = xs
    rng = np.random.default_rng(1)
    for n, bits, hi in ((1, 64, 10), (5000, 64, 1 << 62), (100003, 20, 1 << 20), (70000, 33, 1000)):
        k = rng.integers(0, hi, n, dtype=np.int64).astype(np.uint64)
        if n > 10:
            k[::7] = k[3]                      # duplicates keep input order
        v = np.arange(n, dtype=np.uint32)
        kt = torch.from_numpy(k.view(np.int64)).cuda()
        vt = torch.from_numpy(v.view(np.int32)).cuda()
        grid.radix_sort_pairs(kt, vt, bits)
        order = np.argsort(k, kind="stable")
        assert np.array_equal(kt.cpu().numpy().view(np.uint64), k[order])
        assert np.array_equal(vt.cpu().numpy().view(np.uint32), v[order])


def test_hashset_semantics(xs):
    grid, _, _ = xs
    rng = np.random.default_rng(2)
    hs = grid.VoxelHashSet(1024)
    keys = rng.integers(0, 1 << 62, 50000, dtype=np.int64).astype(np.uint64)
    keys[1000:2000] = keys[:1000]
    new = hs.insert(keys).cpu().numpy()
    seen = set(keys.tolist())
    # parallel insert-if-absent: exactly one occurrence of every distinct key reports "new"
    uniq, inv = np.unique(keys, return_inverse=True)
    assert np.array_equal(np.bincount(inv, weights=new), np.ones(uniq.size))
    assert len(hs) == len(seen)                                   # grew past the initial 1024 slots
    assert not hs.insert(keys[:500]).cpu().numpy().any()          # second insert: nothing new
    probe = np.concatenate([keys[:100], rng.integers(0, 1 << 62, 100, dtype=np.int64).astype(np.uint64)])
    got = hs.contains(probe).cpu().numpy()
    assert np.array_equal(got, np.array([int(p) in seen for p in probe]))


# ------------------------------------------------------------ per-voxel features
# Feature gather rule: supervision.py:133-147 (per-frame (C, Hf, Wf) map,
# nearest lattice cell).  First-pick copies the representative's gathered
# value; mean mode averages the members' values in fp64, pid order
# (oracle/grid.py, np.add.at then / count).

@pytest.mark.parametrize("mode", ["first", "mean"])
@pytest.mark.parametrize("force_sort", ["0", "1"])
@pytest.mark.parametrize("W", [128, 130])          # fused front end (W % 4 == 0) / two-kernel front end
def test_grid_features_match_oracle(xs, mode, force_sort, W):
    import os
    grid, _, synth = xs
    frames, intr4 = _scene(synth, 11, 96, W, 3, spheres=True)
    rng = np.random.default_rng(12)
    feats = rng.normal(size=(3, 16, 24, 33)).astype(np.float32)
    D = np.stack([f[0] for f in frames])
    C = np.stack([f[1] for f in frames])
    R = np.stack([f[2] for f in frames])
    T = np.stack([f[3] for f in frames])
    os.environ["XGS_GRID_SORT"] = force_sort
    try:
        gs = grid.GridSampler(intr4, 0.02, mode=mode)
        warm = og.pack_key(np.array([0, 1]), np.array([0, 0]), np.array([0, 0]))
        gs.occupied.insert(warm)
        got = gs.sample(D, (R, T), C, features=feats).to_numpy()
    finally:
        os.environ.pop("XGS_GRID_SORT", None)
    ref = og.grid_sample(frames, np.array(intr4), 0.02, set(int(k) for k in warm), mode=mode, features=list(feats))
    assert got["feature"].shape == ref["feature"].shape
    assert got["feature"].dtype == (np.float32 if mode == "first" else np.float64)
    for name in ("key", "pid", "mu", "color", "feature"):
        assert np.array_equal(np.asarray(got[name], dtype=ref[name].dtype), ref[name]), name
    if mode == "mean":
        assert np.array_equal(got["count"], ref["count"])


def test_grid_features_device_tensors_and_shape_errors(xs, cuda):
    import torch
    grid, _, synth = xs
    frames, intr4 = _scene(synth, 13, 48, 64, 2)
    feats = np.random.default_rng(14).normal(size=(2, 4, 48, 64)).astype(np.float32)
    D = torch.from_numpy(np.stack([f[0] for f in frames])).cuda()
    R = np.stack([f[2] for f in frames])
    T = np.stack([f[3] for f in frames])
    from paper_2603_09632_b200.errors import InvalidInputError
    gs = grid.GridSampler(intr4, 0.03)
    with pytest.raises(InvalidInputError):       # one map for a two-frame batch
        gs.sample(D, (R, T), features=feats[0])
    with pytest.raises(InvalidInputError):       # wrong frame count
        gs.sample(D, (R, T), features=feats[:1])
    r = gs.sample(D, (R, T), features=torch.from_numpy(feats).cuda())
    assert r.feature.is_cuda and r.feature.shape == (len(r), 4)
    ref = og.grid_sample([(f[0], f[1], f[2], f[3]) for f in frames], np.array(intr4), 0.03, set(),
                         features=list(feats))
    assert np.array_equal(r.feature.cpu().numpy().astype(np.float64), ref["feature"])
    # single-frame batch: a (C, Hf, Wf) map is accepted
    one = grid.GridSampler(intr4, 0.03).sample(D[0], (R[:1], T[:1]), features=feats[0]).to_numpy()
    ref1 = og.grid_sample([frames[0]], np.array(intr4), 0.03, set(), features=[feats[0]])
    assert np.array_equal(one["feature"].astype(np.float64), ref1["feature"])


@pytest.mark.parametrize("n", [1, 2, 7, 100_000, 100_001])
def test_pose_depths_and_median_on_device(xs, n):
    """slam.pose_depths (slam.py:654-655) in the reference's BLAS evaluation
    order (bit-identical to pose.transform(mu)[:, 2]) and np.median of it
    (the densify fallback depth) through the device radix sort."""
    _, slam, _ = xs
    from paper_2603_09632_b200.core import CameraPose, GaussianField
    rng = np.random.default_rng(n)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    if np.linalg.det(Q) < 0:
        Q[:, 0] *= -1
    pose = CameraPose(Q, rng.normal(size=3) * 3)
    mu = rng.normal(size=(n, 3)) * 4
    mu[::13] = mu[0]                        # duplicate depths
    field = GaussianField(mu=mu, quat=np.tile([1.0, 0, 0, 0], (n, 1)), scale=np.full((n, 3), 0.01),
                          opacity=np.full(n, 0.5), color=np.zeros((n, 3)), logits=np.zeros((n, 2)))
    ref = pose.transform(mu)[:, 2]
    assert np.array_equal(slam.pose_depths(field, pose), ref)
    assert slam.median_pose_depth(field, pose) == float(np.median(ref))
