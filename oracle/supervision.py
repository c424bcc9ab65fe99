"""TEST INFRASTRUCTURE ONLY — NumPy restatement of the grid-sampled supervision
targets (reference pkg/src/semsplat/supervision.py), pinned by
tests/golden/supervision.npz (generated from the reference)."""

from __future__ import annotations

import numpy as np

NORM_EPS = 1e-8


def grid_resolution(H, s, o):                          # supervision.py:21-31
    return max(0, 1 + (H - 1 - o) // s)


def lattice(H, W, s, oh, ow):                          # supervision.py:55-67
    rows = oh + s * np.arange(grid_resolution(H, s, oh))
    cols = ow + s * np.arange(grid_resolution(W, s, ow))
    return rows, cols


def target_continuous(P, H, W, s, oh, ow):              # supervision.py:138-147
    rows, cols = lattice(H, W, s, oh, ow)
    uu = np.floor(rows.astype(np.float64) * (P.shape[1] - 1) / max(H - 1, 1) + 0.5).astype(np.int64)
    vv = np.floor(cols.astype(np.float64) * (P.shape[2] - 1) / max(W - 1, 1) + 0.5).astype(np.int64)
    return P[:, uu][:, :, vv], np.ones((1, rows.size, cols.size))


def target_discrete(S, Phi, H, W, s, oh, ow):           # supervision.py:118-130
    rows, cols = lattice(H, W, s, oh, ow)
    r = S[np.ix_(rows, cols)]
    valid = r != -1
    G = np.zeros((Phi.shape[1], rows.size, cols.size))
    if r.size:
        G[:, valid] = Phi[r[valid]].T
    return G, valid[None].astype(np.float64)


def pad(G, V, H, W, s):                                  # supervision.py:208-221
    Hp, Wp = -(-H // s), -(-W // s)
    Gp = np.zeros((G.shape[0], Hp, Wp))
    Vp = np.zeros((1, Hp, Wp))
    Gp[:, :G.shape[1], :G.shape[2]] = G
    Vp[:, :V.shape[1], :V.shape[2]] = V
    return Gp, Vp


def semantic_loss(pred, G, V, lam=1.0):                  # supervision.py:150-184
    mask = V[0] > 0
    n = int(mask.sum())
    if n == 0:
        return 0.0, np.zeros_like(pred)
    D = pred.shape[0]
    p, t = pred[:, mask], G[:, mask]
    np_, nt = np.linalg.norm(p, axis=0), np.linalg.norm(t, axis=0)
    a, b = np_ + NORM_EPS, nt + NORM_EPS
    dot = np.sum(p * t, axis=0)
    cos = dot / (a * b)
    both = (np_ == 0) & (nt == 0)
    cos[both] = 1.0
    l1 = np.sum(np.abs(p - t), axis=0) / D
    loss = lam * (np.mean(1.0 - cos) + np.mean(l1))
    safe = np.where(np_ > 0, np_, 1.0)
    dcos = t / (a * b) - (dot / (safe * a * a * b)) * p * (np_ > 0)
    dcos[:, both] = 0.0
    cot = np.zeros_like(pred)
    cot[:, mask] = lam * (-dcos + np.sign(p - t) / D) / n
    return float(loss), cot


def next_offset(step, s, seed=0):                        # supervision.py:187-202
    if s == 1:
        return (0, 0)
    n = s * s
    cycle, pos = divmod(int(step), n)
    k = int(np.random.default_rng([int(seed), cycle]).permutation(n)[pos])
    return (k // s, k % s)
