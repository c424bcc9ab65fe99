"""TEST INFRASTRUCTURE ONLY — CPU oracle for voxel grid sampling of RGB-D frames.

What follows the reference:
  * back-projection — ``slam.backproject`` (slam.py:594-598) in fp64, reference
    operation order, u = row paired with fx/cx (core.py:5-9); pinned bit-for-bit
    by golden vectors from the reference (tests/golden/backproject.npz);
  * valid-pixel rule ``depth > 0`` (slam.py:626), colour ``rgb/255`` in fp64
    (reference colours are floats in [0,1], world.py:70), new-splat size
    ``max(min_scale, 0.5*s*depth/fx)`` (slam.py:631), emission in row-major
    pixel order (slam.py:621-632), stride lattice (slam.py:621-623,
    supervision.py:21-67) and the pixel->feature gather rule of
    ``build_target_continuous`` (supervision.py:133-147).
What is builder-defined (SURVEY.md §8(a) g8 — no reference code exists, parity
for this part is pinned by hand-computed KATs only):
  * key: ix = floor(p/vs) per axis, 21-bit fields biased by 2^20,
    key = (ix'<<42)|(iy'<<21)|iz'; out-of-range points are dropped;
  * representative: lowest (frame, pixel) id in the voxel ("first"), or the
    sequential pixel-order mean of position/colour/feature over the voxel's
    points in the representative's frame ("mean");
  * incremental: voxels already in the occupied set are rejected; the new
    keys are inserted after the batch;
  * output order: ascending representative (frame, pixel) id.
"""

from __future__ import annotations

import numpy as np

from . import native

KEY_BIAS = 1 << 20
KEY_INVALID = np.uint64(0xFFFFFFFFFFFFFFFF)


def pack_key(ix, iy, iz):
    ix, iy, iz = (np.asarray(a, dtype=np.int64) + KEY_BIAS for a in (ix, iy, iz))
    return ((ix.astype(np.uint64) << np.uint64(42)) | (iy.astype(np.uint64) << np.uint64(21))
            | iz.astype(np.uint64))


def unpack_key(key):
    key = np.asarray(key, dtype=np.uint64)
    m = np.uint64((1 << 21) - 1)
    return tuple(((key >> np.uint64(s)) & m).astype(np.int64) - KEY_BIAS for s in (42, 21, 0))


def feature_gather_index(H, W, Hf, Wf):
    """supervision.py:133-147 nearest-neighbour map, floor(x + 0.5) rounding."""
    u = np.arange(H, dtype=np.float64)
    v = np.arange(W, dtype=np.float64)
    uu = np.floor(u * (Hf - 1) / max(H - 1, 1) + 0.5).astype(np.int64)
    vv = np.floor(v * (Wf - 1) / max(W - 1, 1) + 0.5).astype(np.int64)
    return uu, vv


def grid_sample(frames, intr4, voxel, occupied=None, stride=1, mode="first",
                min_scale=1e-3, features=None):
    """Voxel-grid sample a batch of frames.

    frames:   list of (depth (H,W) float32, color (H,W,3) uint8, R (3,3), t (3,))
    intr4:    (fx, fy, cx, cy), reference convention (u = row pairs fx/cx)
    occupied: set of uint64 keys already in the map (updated in place)
    features: optional list of per-frame (D,Hf,Wf) feature maps
    """
    if occupied is None:
        occupied = set()
    fx = float(intr4[0])
    allk, allp, allpid, allfr, alld, allc = [], [], [], [], [], []
    allf = []
    for f, (depth, color, R, t) in enumerate(frames):
        H, W = depth.shape
        keys, pts = native.grid_keys(depth, intr4, R, t, voxel, stride)
        idx = np.nonzero(keys != KEY_INVALID)[0]
        allk.append(keys[idx])
        allp.append(pts[idx])
        allpid.append(f * H * W + idx)
        allfr.append(np.full(idx.size, f, dtype=np.int64))
        alld.append(depth.reshape(-1)[idx].astype(np.float64))
        allc.append(color.reshape(-1, 3)[idx].astype(np.float64) / 255.0)
        if features is not None:
            P = np.asarray(features[f], dtype=np.float64)
            uu, vv = feature_gather_index(H, W, P.shape[1], P.shape[2])
            allf.append(P[:, uu[idx // W], vv[idx % W]].T)
    keys = np.concatenate(allk)
    pts = np.concatenate(allp)
    pid = np.concatenate(allpid).astype(np.int64)
    fr = np.concatenate(allfr)
    dep = np.concatenate(alld)
    col = np.concatenate(allc)
    feat = np.concatenate(allf) if features is not None else None

    order = np.argsort(keys, kind="stable")  # input is in pid order -> ties by pid
    sk = keys[order]
    head = np.ones(sk.size, dtype=bool)
    head[1:] = sk[1:] != sk[:-1]
    seg = np.cumsum(head) - 1
    heads = order[head]
    occ = np.fromiter(occupied, dtype=np.uint64, count=len(occupied))
    is_new = ~np.isin(keys[heads], occ)
    heads_new = np.sort(heads[is_new])                 # ascending representative pid
    n = heads_new.size

    out = dict(key=keys[heads_new], pid=pid[heads_new], frame=fr[heads_new],
               depth=dep[heads_new])
    scale = np.maximum(min_scale, 0.5 * stride * dep[heads_new] / fx)
    out["scale"] = scale
    if mode == "first":
        out["mu"] = pts[heads_new]
        out["color"] = col[heads_new]
        if feat is not None:
            out["feature"] = feat[heads_new]
    elif mode == "mean":
        # members of a voxel: its points in the representative's frame, summed
        # sequentially in ascending pid order (np.add.at), then / count
        head_of = heads[seg]                      # for sorted position -> head index
        member = order[fr[order] == fr[head_of]]
        mhead = head_of[fr[order] == fr[head_of]]
        slot = np.full(pid.size, -1, dtype=np.int64)
        slot[heads_new] = np.arange(n)
        ms = slot[mhead]
        keep = ms >= 0
        member, ms = member[keep], ms[keep]
        # sequential order inside each voxel = ascending pid = sorted order
        cnt = np.bincount(ms, minlength=n).astype(np.float64)
        for name, arr in (("mu", pts), ("color", col), ("feature", feat)):
            if arr is None:
                continue
            acc = np.zeros((n, arr.shape[1]))
            np.add.at(acc, ms, arr[member])
            out[name] = acc / cnt[:, None]
        out["count"] = cnt
    else:
        raise ValueError(mode)
    occupied.update(int(k) for k in out["key"])
    out["n_valid"] = int(keys.size)
    out["n_voxels"] = int(heads.size)
    return out
