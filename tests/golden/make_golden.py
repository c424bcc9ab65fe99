"""Generate the golden vectors that pin the oracle (and through it the CUDA path).

Runs the REFERENCE itself (semsplat 0.1.0 at /root/reference/pkg/src, imported
read-only) on seeded inputs and stores inputs + outputs as small .npz fixtures.
Only this script reads /root/reference; the fixtures travel with the repo.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from semsplat.core import (CameraIntrinsics, CameraPose, Codebook,  # noqa: E402
                           FeatureReservoir, GaussianField)
from semsplat import slam, vq  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def mixture(rng, n, D, centres, sigma):
    C = rng.normal(size=(centres, D))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    ids = rng.integers(0, centres, n)
    x = C[ids] + sigma * rng.normal(size=(n, D))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(np.float32)


def make_cb(E, lam=0.96, eps=1e-5, cap=64):
    E = np.asarray(E, dtype=float)
    return Codebook(E=E, N=np.zeros(E.shape[0]), M=np.zeros_like(E), lam=lam, epsilon=eps,
                    reservoir=FeatureReservoir(cap, E.shape[1]))


def gen_distances():
    rng = np.random.default_rng(100)
    out = {}
    for D in (1, 3, 7, 8, 9, 17, 100, 128, 129, 255, 512, 768, 1152):
        x = rng.normal(size=(6, D))
        E = rng.normal(size=(5, D))
        out[f"x_{D}"] = x
        out[f"E_{D}"] = E
        out[f"d_{D}"] = vq.squared_distances(x, make_cb(E))
    np.savez_compressed(os.path.join(OUT, "sqdist.npz"), **out)


def gen_assign():
    rng = np.random.default_rng(101)
    out = {}
    # C1-like: K=256, D=512, 64-centre mixture sigma 0.1, E from random rows
    x = mixture(rng, 512, 512, 64, 0.1)
    E = x[rng.choice(512, 256, replace=False)].astype(np.float64)
    out["c1_x"], out["c1_E"] = x, E.astype(np.float32)  # exact: rows of x
    out["c1_codes"] = vq.assign_batch(x, make_cb(E))
    # C2-like subset: K=1024, D=512, 1024-centre sigma 0.05
    x = mixture(rng, 384, 512, 1024, 0.05)
    E = mixture(rng, 512, 512, 1024, 0.05).astype(np.float64)
    out["c2_x"], out["c2_E"] = x, E.astype(np.float32)  # exact upcast
    out["c2_codes"] = vq.assign_batch(x, make_cb(E))
    # exact ties: duplicated codewords and equidistant points -> lowest index
    E = rng.normal(size=(16, 8))
    E[9] = E[3]
    E[12] = E[3]
    xs = np.concatenate([E[[3, 9, 12]], rng.normal(size=(61, 8))])
    out["tie_x"], out["tie_E"] = xs, E
    out["tie_codes"] = vq.assign_batch(xs, make_cb(E))
    E = np.array([[0.0, 0.0], [2.0, 0.0], [1.0, 1.0], [1.0, -1.0]])
    xs = np.array([[1.0, 0.0], [0.5, 0.5], [3.0, 0.0], [-1.0, 0.0]])
    out["tie2_x"], out["tie2_E"] = xs, E
    out["tie2_codes"] = vq.assign_batch(xs, make_cb(E))
    np.savez_compressed(os.path.join(OUT, "assign.npz"), **out)


def gen_accumulate_ema():
    rng = np.random.default_rng(102)
    out = {}
    x = mixture(rng, 2000, 64, 16, 0.1)
    E = x[:32].astype(np.float64) + 0.01
    cb = make_cb(E, lam=0.99)
    st = vq.accumulate(x, cb)
    out["x"], out["E"] = x, E
    out["counts"], out["sums"] = st.counts, st.sums
    cb.N[:] = rng.uniform(0, 5, 32)
    cb.M[:] = rng.normal(size=(32, 64))
    out["N0"], out["M0"] = cb.N.copy(), cb.M.copy()
    e = vq.ema_step(cb, st)
    out["N1"], out["M1"], out["E1"] = e.N, e.M, e.E
    np.savez_compressed(os.path.join(OUT, "accumulate.npz"), **out)


def gen_online():
    out = {}
    # (a) confidence path active (gamma=0.5, tau=0.7): small clustered stream
    rng = np.random.default_rng(103)
    centres = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]])
    cfg = vq.VqConfig(K=4, lam=0.8, gamma=0.5, tau_warm=0.7, delta_dead=1e-2)
    batches = [centres[rng.integers(0, 4, 64)] + rng.normal(0, 0.05, (64, 3)) for _ in range(12)]
    batches += [centres[rng.integers(0, 3, 64)] + rng.normal(0, 0.05, (64, 3)) for _ in range(40)]
    batches += [np.concatenate([centres[rng.integers(0, 4, 60)] + rng.normal(0, 0.05, (60, 3)),
                                rng.uniform(-3, 3, (4, 3))]) for _ in range(20)]
    E0 = centres + 0.1
    cb = make_cb(E0, lam=0.8, cap=128)
    rrng = np.random.default_rng(7)
    Es, Ns, Ms, rev = [], [], [], []
    for b in batches:
        cb, res = vq.online_step(cb, b, cfg, rrng)
        Es.append(cb.E)
        Ns.append(cb.N)
        Ms.append(cb.M)
        rev.append(len(res.revived))
    out["a_batches"] = np.stack(batches)
    out["a_E0"] = E0
    out["a_E"], out["a_N"], out["a_M"] = np.stack(Es), np.stack(Ns), np.stack(Ms)
    out["a_nrev"] = np.array(rev)
    # (b) BASELINE-style: gamma = 0.5/K (mask all-true), lam 0.99, delta 1e-3
    rng = np.random.default_rng(104)
    K, D, n = 64, 32, 256
    x = mixture(rng, n * 8, D, 48, 0.05)
    E0 = x[rng.choice(x.shape[0], K, replace=False)].astype(np.float64)
    cfg = vq.VqConfig(K=K, lam=0.99, gamma=0.5 / K, delta_dead=1e-3)
    cb = make_cb(E0, lam=0.99, cap=300)
    rrng = np.random.default_rng(12)
    Es, Ns, rev = [], [], []
    for i in range(8):
        cb, res = vq.online_step(cb, x[i * n:(i + 1) * n], cfg, rrng)
        Es.append(cb.E)
        Ns.append(cb.N)
        rev.append(len(res.revived))
    out["b_x"], out["b_E0"] = x, E0
    out["b_E"], out["b_N"], out["b_nrev"] = np.stack(Es), np.stack(Ns), np.array(rev)
    # (c) confidence scores / mask values
    rng = np.random.default_rng(105)
    E = rng.normal(size=(7, 5))
    xs = rng.normal(size=(40, 5))
    cbc = make_cb(E)
    out["c_x"], out["c_E"] = xs, E
    out["c_p"] = vq.confidence_scores(xs, cbc, 0.7)
    out["c_mask"] = vq.confidence_mask(xs, cbc, vq.VqConfig(K=7, gamma=0.4))
    # (d) warm start + farthest point seeding
    rng = np.random.default_rng(106)
    buf = rng.normal(size=(50, 3))
    seeds = vq.seed_from_samples(buf, 4)
    ws = vq.warm_start(buf, make_cb(seeds), vq.VqConfig(K=4, gamma=0.3))
    out["d_buf"], out["d_seeds"] = buf, seeds
    out["d_E"], out["d_N"], out["d_used"] = ws.codebook.E, ws.codebook.N, np.array(ws.used)
    np.savez_compressed(os.path.join(OUT, "online.npz"), **out)


def gen_backproject():
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(107)
    n = 12000
    R = Rotation.random(16, random_state=3).as_matrix()
    t = rng.normal(size=(16, 3))
    intr = CameraIntrinsics(fx=525.0, fy=525.0, cx=239.5, cy=319.5, height=480, width=640)
    pose_id = rng.integers(0, 16, n)
    u = rng.integers(0, 480, n)
    v = rng.integers(0, 640, n)
    d = rng.uniform(0.3, 8.0, n).astype(np.float32)
    p = np.empty((n, 3))
    for i in range(n):
        pose = CameraPose(R[pose_id[i]], t[pose_id[i]])
        p[i] = slam.backproject(pose, intr, int(u[i]), int(v[i]), float(d[i]))
    np.savez_compressed(os.path.join(OUT, "backproject.npz"), R=R, t=t,
                        intr=np.array([525.0, 525.0, 239.5, 319.5]), pose_id=pose_id,
                        u=u, v=v, d=d, p=p)


def gen_densify():
    """densify_and_prune on an EMPTY field (coverage alpha == 0, no render):
    every stride-4 lattice pixel is inserted (slam.py:601-651)."""
    from semsplat.world import CameraFrame
    rng = np.random.default_rng(108)
    H, W = 24, 32
    depth = rng.uniform(0.5, 5.0, (H, W)).astype(np.float32)
    depth[rng.random((H, W)) < 0.2] = 0.0
    color = rng.random((3, H, W))
    from scipy.spatial.transform import Rotation
    pose = CameraPose(Rotation.random(random_state=5).as_matrix(), rng.normal(size=3))
    frame = CameraFrame(frame_id=0, pose=pose, color=color, depth=depth)
    win = slam.KeyframeWindow(4)
    win.insert(frame, pose)
    empty = GaussianField(mu=np.zeros((0, 3)), quat=np.zeros((0, 4)), scale=np.zeros((0, 3)),
                          opacity=np.zeros(0), color=np.zeros((0, 3)), logits=np.zeros((0, 5)))
    cfg = slam.SlamConfig()
    out = slam.densify_and_prune(empty, win, cfg, K=5)
    # non-empty map: the empty-map splats (some pruned, some re-weighted) seen
    # from a nearby second keyframe -> render-coverage skipping (slam.py:610-626)
    op = out.opacity.copy()
    op[::7] = 0.005                                     # pruned
    op[1::3] = rng.uniform(0.2, 0.95, op[1::3].size)
    field1 = GaussianField(mu=out.mu, quat=out.quat, scale=out.scale * 1.5, opacity=op, color=out.color,
                           logits=out.logits, generation=out.generation)
    from scipy.spatial.transform import Rotation as Rt
    pose2 = CameraPose(Rt.from_rotvec([0.02, -0.03, 0.01]).as_matrix() @ pose.rotation,
                       pose.translation + np.array([0.05, 0.0, -0.03]))
    depth2 = rng.uniform(0.5, 5.0, (H, W)).astype(np.float32)
    depth2[rng.random((H, W)) < 0.2] = 0.0
    frame2 = CameraFrame(frame_id=1, pose=pose2, color=rng.random((3, H, W)), depth=depth2)
    win2 = slam.KeyframeWindow(4)
    win2.insert(frame2, pose2)
    out2 = slam.densify_and_prune(field1, win2, cfg, K=5)
    np.savez_compressed(os.path.join(OUT, "densify.npz"), depth=depth, color=color,
                        R=pose.rotation, t=pose.translation, mu=out.mu, scale=out.scale,
                        col=out.color, opacity=out.opacity, quat=out.quat,
                        generation=np.array(out.generation),
                        f1_mu=field1.mu, f1_quat=field1.quat, f1_scale=field1.scale, f1_opacity=field1.opacity,
                        f1_color=field1.color, f1_logits=field1.logits, R2=pose2.rotation, t2=pose2.translation,
                        depth2=depth2, color2=frame2.color, m2_mu=out2.mu, m2_scale=out2.scale,
                        m2_color=out2.color, m2_opacity=out2.opacity, m2_generation=np.array(out2.generation))


def gen_supervision():
    """supervision.py:21-221 — lattice, continuous / discrete targets, loss + cotangent,
    offset schedule, padding."""
    from semsplat import supervision as sup
    rng = np.random.default_rng(109)
    out = {}
    H, W = 37, 53
    P = rng.normal(size=(6, 5, 7))
    S = rng.integers(-1, 4, (H, W))
    Phi = rng.normal(size=(4, 6))
    src = sup.ContinuousFeatureSource(P)
    ann = sup.RegionAnnotation(S, Phi)
    out["P"], out["S"], out["Phi"] = P, S, Phi
    cases = [(1, 0, 0), (2, 1, 0), (3, 2, 1), (4, 3, 3), (5, 0, 4)]
    for i, (s_, oh, ow) in enumerate(cases):
        g = sup.GridSpec(H, W, s_, oh, ow)
        tc = sup.build_target_continuous(src, g)
        td = sup.build_target_discrete(ann, g)
        out[f"cont_G_{i}"], out[f"disc_G_{i}"], out[f"disc_V_{i}"] = tc.G_star, td.G_star, td.V
        pt = sup.pad_target(td, g)
        out[f"pad_G_{i}"], out[f"pad_V_{i}"] = pt.G_star, pt.V
        pred = rng.normal(size=td.G_star.shape)
        pred[:, 0, 0] = 0.0
        loss, cot = sup.masked_semantic_loss(pred, td, lambda_sem=0.7)
        out[f"pred_{i}"], out[f"loss_{i}"], out[f"cot_{i}"] = pred, np.array(loss), cot
    out["cases"] = np.array(cases)
    out["offsets"] = np.array([sup.next_offset(k, 4, 3) for k in range(40)])
    out["offsets_s1"] = np.array([sup.next_offset(k, 1, 3) for k in range(3)])
    np.savez_compressed(os.path.join(OUT, "supervision.npz"), **out)


def gen_thinker():
    """core.mixture_weights / softmax_vjp / decode_feature and thinker.* (§8(f) #3)."""
    from semsplat import thinker
    from semsplat.core import decode_feature, mixture_weights, softmax_vjp
    rng = np.random.default_rng(400)
    out = {}
    for tag, (n, K, D) in {"a": (300, 37, 24), "b": (129, 256, 64)}.items():
        L = rng.normal(scale=3.0, size=(n, K))
        L[0] = 0.0                            # uniform row: maximum entropy
        L[1] = L[2]                           # duplicate rows: entropy ties -> lower index first
        L[3, 5] = 40.0                        # near one-hot
        L[4] = L[7]
        E = rng.normal(size=(K, D))
        up = rng.normal(size=(n, K))
        cb = make_cb(E)
        out[f"{tag}_L"], out[f"{tag}_E"], out[f"{tag}_up"] = L, E, up
        out[f"{tag}_w"] = mixture_weights(L)
        out[f"{tag}_vjp"] = softmax_vjp(L, up)
        out[f"{tag}_dec"] = decode_feature(L, cb)
        out[f"{tag}_dec1"] = decode_feature(L[5], cb)
        out[f"{tag}_H"] = thinker.semantic_entropy(L)
        field = GaussianField(mu=np.zeros((n, 3)), quat=np.tile([1.0, 0, 0, 0], (n, 1)), scale=np.ones((n, 3)),
                              opacity=np.ones(n), color=np.zeros((n, 3)), logits=L)
        enc = thinker.StubTextEncoder(D, region_table=E[:6])
        q = thinker.TextQuery.from_prompt("region:2", enc)
        out[f"{tag}_qpos"], out[f"{tag}_qneg"] = q.positive, np.stack(q.negatives)
        out[f"{tag}_rel"] = thinker.relevance_per_gaussian(field, cb, q)
        res = thinker.query_field(field, cb, q)
        out[f"{tag}_mask"], out[f"{tag}_fallback"] = res.mask, np.array(res.fallback_used)
        m2, fb2 = thinker.mask_gaussians(out[f"{tag}_rel"], 0.999999, fallback_frac=0.05)
        out[f"{tag}_mask_fb"], out[f"{tag}_fb2"] = m2, np.array(fb2)
        ts = thinker.sample_tokens(field, cb, 17)
        out[f"{tag}_tok_idx"], out[f"{tag}_tok_H"], out[f"{tag}_tok_F"] = ts.indices, ts.entropies, ts.features
        ts2 = thinker.sample_tokens(field, cb, n + 5)
        out[f"{tag}_tok2_idx"], out[f"{tag}_tok2_clamped"] = ts2.indices, np.array(ts2.clamped)
        W = rng.random(size=(K, 5, 7))
        out[f"{tag}_wmap"] = W
        out[f"{tag}_relpix"] = thinker.relevance_per_pixel([type("M", (), {"data": W})()], [cb], q)
    out["neg_phrases_vecs"] = np.stack(thinker.StubTextEncoder(24).negatives())
    out["hash_vec"] = thinker.StubTextEncoder(24).encode("a lamp")
    np.savez_compressed(os.path.join(OUT, "thinker.npz"), **out)


def raster_scene(rng, n, H, W, K=6, D=5):
    from semsplat.core import rot_to_quat
    mu = np.column_stack([rng.uniform(-1.5, 1.5, n), rng.uniform(-1.5, 1.5, n), rng.uniform(-0.5, 4.0, n)])
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scale = np.exp(rng.uniform(np.log(0.01), np.log(0.3), (n, 3)))
    opacity = rng.uniform(0.05, 1.0, n)
    opacity[: n // 10] = 0.999                     # near-opaque splats: early termination
    color = rng.random((n, 3))
    logits = rng.normal(size=(n, K))
    field = GaussianField(mu=mu, quat=q, scale=scale, opacity=opacity, color=color, logits=logits)
    ang = rng.normal(scale=0.1, size=3)
    c, s_ = np.cos(ang), np.sin(ang)
    Rz = np.array([[c[2], -s_[2], 0], [s_[2], c[2], 0], [0, 0, 1]])
    Rx = np.array([[1, 0, 0], [0, c[0], -s_[0]], [0, s_[0], c[0]]])
    pose = CameraPose(Rz @ Rx, np.array([0.05, -0.1, 1.2]))
    intr = CameraIntrinsics(fx=0.9 * W, fy=0.85 * W, cx=(H - 1) / 2 + 0.3, cy=(W - 1) / 2 - 0.2, height=H, width=W)
    E = rng.normal(size=(K, D))
    return field, pose, intr, E


def gen_raster():
    """rasterizer.build_blend_pairs / render / render_channels_grid / argmax /
    feature_gradients on seeded scenes (dense all-pairs path and the
    per-Gaussian bounding-box path of the reference)."""
    from semsplat import rasterizer as rz
    from semsplat.supervision import GridSpec
    rng = np.random.default_rng(500)
    out = {}
    for tag, (n, H, W, s, oh, ow) in {"dense": (150, 24, 32, 1, 0, 0), "bbox": (1200, 24, 44, 1, 0, 0),
                                       "grid": (1200, 24, 44, 3, 1, 2)}.items():
        field, pose, intr, E = raster_scene(rng, n, H, W)
        for k in ("mu", "quat", "scale", "opacity", "color", "logits"):
            out[f"{tag}_{k}"] = getattr(field, k)
        out[f"{tag}_R"], out[f"{tag}_t"], out[f"{tag}_E"] = pose.rotation, pose.translation, E
        out[f"{tag}_intr"] = np.array([intr.fx, intr.fy, intr.cx, intr.cy, H, W, intr.near, intr.far])
        grid = GridSpec(H=H, W=W, s=s, o_h=oh, o_w=ow)
        out[f"{tag}_grid"] = np.array([H, W, s, oh, ow])
        bp = rz.build_blend_pairs(field, pose, intr, grid.rows(), grid.cols())
        for k in ("gauss", "pixel", "weight", "alpha_prime", "t_before", "alive", "depth"):
            out[f"{tag}_bp_{k}"] = getattr(bp, k)
        out[f"{tag}_bp_steps"] = np.array(bp.blend_steps)
        if s == 1:
            r = rz.render(field, pose, intr)
            out[f"{tag}_r_color"], out[f"{tag}_r_depth"], out[f"{tag}_r_alpha"] = r.color, r.depth, r.alpha
            out[f"{tag}_steps"] = np.array(r.blend_steps)
            out[f"{tag}_argmax"] = rz.render_argmax_ids(field, pose, intr)
        payload = rng.normal(size=(n, 4))
        out[f"{tag}_payload"] = payload
        out[f"{tag}_chan"] = rz.render_channels_grid(field, payload, pose, intr, grid).data
        cb = make_cb(E)
        up = rng.normal(size=(E.shape[1], grid.H_s, grid.W_s))
        out[f"{tag}_up"] = up
        fgr = rz.feature_gradients(field, cb, pose, intr, grid, up)
        out[f"{tag}_fg"], out[f"{tag}_lg"] = fgr.feature_grads, fgr.logit_grads
        out[f"{tag}_feat"] = rz.render_features_grid(field, cb, pose, intr, grid).data
    np.savez_compressed(os.path.join(OUT, "raster.npz"), **out)


GENERATORS = {"supervision": gen_supervision, "distances": gen_distances, "assign": gen_assign,
              "accumulate": gen_accumulate_ema, "online": gen_online, "backproject": gen_backproject,
              "densify": gen_densify, "thinker": gen_thinker,
              "raster": gen_raster}

if __name__ == "__main__":
    for name in (sys.argv[1:] or list(GENERATORS)):
        GENERATORS[name]()
    for f in sorted(os.listdir(OUT)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(OUT, f)))
