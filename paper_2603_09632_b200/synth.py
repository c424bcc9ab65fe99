"""Seeded synthetic inputs with the BASELINE.json shapes (configs C1-C5).

The paper's TUM RGB-D sequence and VFM features are not available offline;
these generators stand in for them: depth frames
ray-cast against random planes (+ spheres), Gaussian depth noise, a fraction of
zero (invalid) pixels, uniform uint8 colour, circular / random-walk camera
trajectories, and unit-norm features from a Gaussian mixture.  Host NumPy,
generated once outside any timed region.
"""

from __future__ import annotations

import numpy as np

from .core import CameraPose


def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> CameraPose:
    """World->camera pose whose optical axis (+z) points from eye to target;
    camera x (rows, u) points down, y (columns, v) right."""
    eye, target, up = (np.asarray(a, dtype=np.float64) for a in (eye, target, up))
    z = target - eye
    z /= np.linalg.norm(z)
    y = np.cross(z, up)
    if np.linalg.norm(y) < 1e-9:
        y = np.cross(z, [1.0, 0.0, 0.0])
    y /= np.linalg.norm(y)
    x = np.cross(y, z)
    R = np.stack([x, y, z])           # rows: camera axes in world coordinates
    if np.linalg.det(R) < 0:
        R[0] = -R[0]
    return CameraPose(R, -R @ eye)


def circle_trajectory(n, radius=2.0, step_deg=5.0, height=0.0):
    poses = []
    for i in range(n):
        a = np.deg2rad(step_deg * i)
        eye = np.array([radius * np.cos(a), radius * np.sin(a), height])
        poses.append(look_at(eye, np.zeros(3)))
    return poses


def random_walk_trajectory(n, rng, step_t=0.01, step_deg=1.0):
    poses = [CameraPose(np.eye(3), np.zeros(3))]
    for _ in range(n - 1):
        w = rng.normal(0, np.deg2rad(step_deg), 3)
        th = np.linalg.norm(w)
        k = w / th if th > 0 else np.zeros(3)
        Kx = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
        dR = np.eye(3) + np.sin(th) * Kx + (1 - np.cos(th)) * Kx @ Kx
        p = poses[-1]
        R = dR @ p.rotation
        U, _, Vt = np.linalg.svd(R)
        R = U @ Vt
        poses.append(CameraPose(R, p.translation + rng.normal(0, step_t, 3)))
    return poses


def random_planes(rng, n, centre=np.zeros(3), spread=3.0):
    planes = []
    for _ in range(n):
        nrm = rng.normal(size=3)
        nrm /= np.linalg.norm(nrm)
        pt = centre + rng.uniform(-spread, spread, 3)
        planes.append((nrm, float(nrm @ pt)))
    return planes


def facing_planes(rng, n, dmin=3.0, dmax=7.0, tilt=0.3):
    """n walls roughly facing a camera at the origin looking down +z (normal
    ~ +z tilted by N(0, tilt) per axis) at distances U(dmin, dmax)."""
    planes = []
    for _ in range(n):
        nrm = np.array([rng.normal(0, tilt), rng.normal(0, tilt), 1.0])
        nrm /= np.linalg.norm(nrm)
        planes.append((nrm, float(rng.uniform(dmin, dmax))))
    return planes


def render_depth(pose, intr4, H, W, planes=(), spheres=(), dmin=0.3, dmax=8.0):
    """Camera-z depth of the first surface hit; 0 where nothing is hit in range."""
    fx, fy, cx, cy = intr4
    u, v = np.meshgrid(np.arange(H, dtype=np.float64), np.arange(W, dtype=np.float64), indexing="ij")
    dcam = np.stack([(u - cx) / fx, (v - cy) / fy, np.ones_like(u)], axis=-1)   # z = 1 -> t == depth
    R, t = pose.rotation, pose.translation
    dw = dcam @ R                      # R^T d for every pixel
    C = -R.T @ t
    best = np.full((H, W), np.inf)
    for nrm, c in planes:
        den = dw @ nrm
        with np.errstate(divide="ignore", invalid="ignore"):
            tt = (c - nrm @ C) / den
        tt[(tt <= 0) | ~np.isfinite(tt)] = np.inf
        best = np.minimum(best, tt)
    for centre, rad in spheres:
        oc = C - centre
        a = np.sum(dw * dw, axis=-1)
        b = 2 * (dw @ oc)
        cc = oc @ oc - rad * rad
        disc = b * b - 4 * a * cc
        with np.errstate(invalid="ignore"):
            tt = (-b - np.sqrt(disc)) / (2 * a)
        tt[(disc < 0) | (tt <= 0)] = np.inf
        best = np.minimum(best, tt)
    best[(best < dmin) | (best > dmax)] = 0.0
    return best


def render_depth_torch(torch, R, t, intr4, H, W, planes=(), spheres=(), dmin=0.3, dmax=8.0, device="cuda"):
    """render_depth on the device (fp64): R, t fp64 tensors of one world->camera pose."""
    fx, fy, cx, cy = intr4
    f64 = torch.float64
    u = torch.arange(H, device=device, dtype=f64)[:, None].expand(H, W)
    v = torch.arange(W, device=device, dtype=f64)[None, :].expand(H, W)
    dcam = torch.stack([(u - cx) / fx, (v - cy) / fy, torch.ones_like(u)], dim=-1)
    dw = dcam @ R                      # R^T d for every pixel
    C = -(R.T @ t)
    inf = torch.full((H, W), float("inf"), device=device, dtype=f64)
    best = inf.clone()
    for nrm, c in planes:
        n = torch.as_tensor(nrm, device=device, dtype=f64)
        den = dw @ n
        tt = (float(c) - n @ C) / den
        best = torch.minimum(best, torch.where((tt > 0) & torch.isfinite(tt), tt, inf))
    for centre, rad in spheres:
        oc = C - torch.as_tensor(centre, device=device, dtype=f64)
        a = (dw * dw).sum(-1)
        b = 2 * (dw @ oc)
        cc = oc @ oc - rad * rad
        disc = b * b - 4 * a * cc
        tt = (-b - torch.sqrt(torch.clamp(disc, min=0))) / (2 * a)
        best = torch.minimum(best, torch.where((disc >= 0) & (tt > 0), tt, inf))
    return torch.where((best >= dmin) & (best <= dmax), best, torch.zeros_like(best))


def rgbd_frame(rng, pose, intr4, H, W, planes=(), spheres=(), dmin=0.3, dmax=8.0, noise=0.005, zero_frac=0.05,
               clip=None):
    d = render_depth(pose, intr4, H, W, planes, spheres, dmin, dmax)
    valid = d > 0
    d = d + noise * rng.normal(size=d.shape)
    if clip is not None:
        d = np.clip(d, *clip)
    d[~valid] = 0.0
    d[rng.random(d.shape) < zero_frac] = 0.0
    color = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    return d.astype(np.float32), color


def mixture_features(rng, n, D, centres, sigma, dtype=np.float32, C=None):
    if C is None:
        C = rng.normal(size=(centres, D))
        C /= np.linalg.norm(C, axis=1, keepdims=True)
    x = C[rng.integers(0, C.shape[0], n)] + sigma * rng.normal(size=(n, D))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    return x.astype(dtype)


def config1_frame(seed=0):
    """C1: 480x640, 6 planes, 0.5-5 m, sigma 5 mm, 5% zeros, fx=fy=525,
    column centre 319.5 / row centre 239.5 (reference cx <-> rows), identity pose."""
    rng = np.random.default_rng(seed)
    intr4 = (525.0, 525.0, 239.5, 319.5)
    pose = CameraPose.identity()
    planes = random_planes(rng, 6, centre=np.array([0.0, 0.0, 3.0]), spread=2.0)
    d, col = rgbd_frame(rng, pose, intr4, 480, 640, planes=planes, dmin=0.5, dmax=5.0, noise=0.005,
                        zero_frac=0.05, clip=(0.5, 5.0))
    return d, col, pose, intr4
