"""TEST INFRASTRUCTURE ONLY — NumPy restatement of the lattice rasterizer
(reference pkg/src/semsplat/rasterizer.py:89-335 with core.py:40-55,
:402-448), pinned by tests/golden/raster.npz (generated from the reference).
All-pairs evaluation in Gaussian chunks (the reference's dense path; its
bounding-box path selects the same pairs)."""

from __future__ import annotations

import numpy as np

LOG_T_MIN = -69.07755278982137


def quat_to_rot(q):                                              # core.py:40-55
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((q.shape[0], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def screen_cov(mu, quat, scale, Rw, t, fx, fy, cam, eig_floor=0.3):   # core.py:402-448
    R = quat_to_rot(quat)
    sigma = np.einsum("nij,nj,nkj->nik", R, scale ** 2, R)
    x, y, z = cam[:, 0], cam[:, 1], cam[:, 2]
    J = np.zeros((cam.shape[0], 2, 3))
    J[:, 0, 0] = fx / z
    J[:, 0, 2] = -fx * x / z ** 2
    J[:, 1, 1] = fy / z
    J[:, 1, 2] = -fy * y / z ** 2
    JW = J @ Rw
    c2 = np.einsum("nij,njk,nlk->nil", JW, sigma, JW)
    c2 = 0.5 * (c2 + np.swapaxes(c2, 1, 2))
    a, b, c = c2[:, 0, 0], c2[:, 0, 1], c2[:, 1, 1]
    ht = 0.5 * (a + c)
    disc = np.sqrt(np.maximum((0.5 * (a - c)) ** 2 + b * b, 0.0))
    l1, l2 = np.maximum(ht + disc, eig_floor), np.maximum(ht - disc, eig_floor)
    th = 0.5 * np.arctan2(2 * b, a - c)
    ct, st = np.cos(th), np.sin(th)
    return l1 * ct * ct + l2 * st * st, (l1 - l2) * ct * st, l1 * st * st + l2 * ct * ct


def blend_pairs(mu, quat, scale, opacity, Rw, t, intr, rows, cols, term=1e-4, cutoff=3.0, eig_floor=0.3):
    """rasterizer.py:89-191 -> (gauss, pixel, weight, alpha', T_before, alive, depth)."""
    fx, fy, cx, cy, near, far = intr
    cam = mu @ Rw.T + t
    z = cam[:, 2]
    idx = np.nonzero((z > near) & (z < far))[0]
    e = (np.zeros(0, np.int64),) * 2 + (np.zeros(0),) * 3 + (np.zeros(0, bool), np.zeros(0))
    if idx.size == 0:
        return e
    order = idx[np.argsort(z[idx], kind="stable")]
    zs = z[order]
    uc = fx * cam[order, 0] / zs + cx
    vc = fy * cam[order, 1] / zs + cy
    a, b, c = screen_cov(mu[order], quat[order], scale[order], Rw, t, fx, fy, cam[order], eig_floor)
    det = a * c - b * b
    ia, ib, ic = c / det, -b / det, a / det
    uu, vv = np.meshgrid(rows.astype(np.float64), cols.astype(np.float64), indexing="ij")
    uu, vv = uu.ravel(), vv.ravel()
    gi, pi, qk = [], [], []
    for k0 in range(0, order.size, 256):
        sl = slice(k0, k0 + 256)
        du = uu[None, :] - uc[sl, None]
        dv = vv[None, :] - vc[sl, None]
        quad = ia[sl, None] * du * du + 2 * ib[sl, None] * du * dv + ic[sl, None] * dv * dv
        g_, p_ = np.nonzero(quad <= cutoff ** 2)
        gi.append(g_ + k0)
        pi.append(p_)
        qk.append(quad[g_, p_])
    gi, pi, qk = np.concatenate(gi), np.concatenate(pi), np.concatenate(qk)
    if gi.size == 0:
        return e
    ap = opacity[order][gi] * np.exp(-0.5 * qk)
    o = np.argsort(pi, kind="stable")
    pi, gi, ap = pi[o], gi[o], ap[o]
    with np.errstate(divide="ignore"):
        lt = np.maximum(np.log1p(-ap), LOG_T_MIN)
    cs = np.cumsum(lt)
    new = np.empty(pi.size, bool)
    new[0] = True
    new[1:] = pi[1:] != pi[:-1]
    st = np.nonzero(new)[0]
    base = (cs[st] - lt[st])[np.cumsum(new) - 1]
    T = np.exp(cs - lt - base)
    alive = T >= term
    return order[gi], pi, np.where(alive, ap * T, 0.0), ap, T, alive, zs[gi]


def accumulate(gauss, pixel, weight, payload, n_pixels):         # rasterizer.py:194-201
    return np.stack([np.bincount(pixel, weights=weight * payload[gauss, ch], minlength=n_pixels)
                     for ch in range(payload.shape[1])])
