"""Drop-ins for the back-projection / insertion part of ``semsplat.slam``.

``backproject`` (slam.py:594-598) and ``densify_and_prune`` (slam.py:601-651)
keep their reference signatures; the arithmetic runs in libxgs
(``xgs_backproject``: fp64, reference operation order, bit-identical).
``densify_and_prune`` reproduces the reference exactly: on a non-empty map
the coverage test renders the field with the GPU rasterizer
(``rasterizer.render``, slam.py:608-626) and the median fallback depth comes
from ``xgs_pose_depths`` + the in-house radix sort (slam.py:611-613, 654-655).
Passing ``occupied`` / ``voxel_size`` selects the voxel-occupancy variant
instead of the render.  The voxel-grid sampler for
whole RGB-D frames is :class:`grid.GridSampler`.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as nat
from .core import CameraIntrinsics, CameraPose, GaussianField
from .errors import InvalidInputError


@dataclass
class SlamConfig:
    """The densify/prune fields of the reference SlamConfig (slam.py:36-76)."""

    raster: object = None    # rasterizer.RasterConfig (None -> DEFAULT_RASTER), slam.py:76
    min_scale: float = 1e-3
    prune_opacity: float = 0.01
    coverage_alpha: float = 0.5
    insert_stride: int = 4
    insert_opacity: float = 0.8
    default_depth: float = 2.0


@dataclass
class CameraFrame:
    """world.py:67-73 (colour (3,H,W) floats in [0,1], depth (H,W) or None)."""

    frame_id: int
    pose: CameraPose
    color: np.ndarray
    depth: Optional[np.ndarray]


@dataclass
class Keyframe:
    frame: object
    pose: CameraPose


class KeyframeWindow:
    """Sliding keyframe window (slam.py:92-117)."""

    def __init__(self, capacity: int):
        if capacity < 1:
            raise InvalidInputError("window capacity must be >= 1")
        self.capacity = capacity
        self.frames: list = []
        self.log: list = []

    def __len__(self):
        return len(self.frames)

    @property
    def newest(self):
        return self.frames[-1]

    def insert(self, frame, pose):
        self.frames.append(Keyframe(frame=frame, pose=pose))
        self.log.append((frame.frame_id, "insert"))
        if len(self.frames) > self.capacity:
            ev = self.frames.pop(0)
            self.log.append((ev.frame.frame_id, "evict"))
            return ev.frame.frame_id
        return None


def frame_intrinsics(frame, cfg=None, fov_deg: float = 60.0) -> CameraIntrinsics:
    """slam.py:276-286: intrinsics from the frame resolution (60 deg FOV)."""
    H, W = frame.color.shape[1:]
    return CameraIntrinsics.from_fov(H, W, fov_deg)


def backproject_pixels(pose: CameraPose, intr, u, v, depth):
    """Batched slam.backproject: (n,) rows u, columns v, depths -> (n, 3) fp64."""
    t = nat.require_cuda()
    fx, fy, cx, cy = ((intr.fx, intr.fy, intr.cx, intr.cy) if hasattr(intr, "fx")   # ours or the reference's
                      else tuple(float(x) for x in intr))
    host = not any(hasattr(a, "data_ptr") for a in (u, v, depth))
    dev = lambda a: (a if hasattr(a, "data_ptr") else t.from_numpy(np.ascontiguousarray(
        np.asarray(a, dtype=np.float64).reshape(-1)))).to(device="cuda", dtype=t.float64).contiguous()
    U, V, Dd = dev(u), dev(v), dev(depth)
    n = int(U.numel())
    if V.numel() != n or Dd.numel() != n:
        raise InvalidInputError("u, v and depth must have the same length")
    R = t.from_numpy(np.ascontiguousarray(pose.rotation, dtype=np.float64)).to("cuda")
    tr = t.from_numpy(np.ascontiguousarray(pose.translation, dtype=np.float64)).to("cuda")
    out = t.empty((n, 3), dtype=t.float64, device="cuda")
    intr4 = (ctypes.c_double * 4)(fx, fy, cx, cy)   # host array (xgs.h)
    nat.call("xgs_backproject", nat.ptr(R), nat.ptr(tr), intr4, nat.ptr(U), nat.ptr(V), nat.ptr(Dd), n,
             nat.ptr(out), nat.stream_ptr())
    return out.cpu().numpy() if host else out


def backproject(pose: CameraPose, intr: CameraIntrinsics, u: float, v: float, depth: float) -> np.ndarray:
    """slam.py:594-598 — one pixel, bit-identical to the reference."""
    return backproject_pixels(pose, intr, [u], [v], [depth])[0]


def _pose_depths_dev(mu, pose, with_keys=False):
    t = nat.require_cuda()
    M = mu if hasattr(mu, "data_ptr") else t.from_numpy(np.ascontiguousarray(np.asarray(mu, dtype=np.float64)))
    M = M.to(device="cuda", dtype=t.float64).reshape(-1, 3).contiguous()
    n = int(M.shape[0])
    z = t.empty(n, dtype=t.float64, device="cuda")
    key = t.empty(n, dtype=t.int64, device="cuda") if with_keys else None
    idx = t.empty(n, dtype=t.int32, device="cuda") if with_keys else None
    R9 = (ctypes.c_double * 9)(*np.asarray(pose.rotation, dtype=np.float64).reshape(-1))
    t3 = (ctypes.c_double * 3)(*np.asarray(pose.translation, dtype=np.float64).reshape(-1))
    nat.call("xgs_pose_depths", nat.ptr(M), n, R9, t3, nat.ptr(z), nat.ptr(key), nat.ptr(idx), nat.stream_ptr())
    return z, key, idx


def pose_depths(field_: GaussianField, pose: CameraPose):
    """slam.py:654-655 — camera z of every Gaussian centre (device kernel, the
    reference's BLAS evaluation order; NumPy in -> NumPy out)."""
    mu = field_.mu
    z, _, _ = _pose_depths_dev(mu, pose)
    return z if hasattr(mu, "data_ptr") else z.cpu().numpy()


def median_pose_depth(field_: GaussianField, pose: CameraPose) -> float:
    """np.median(pose_depths(field_, pose)) (slam.py:611-613) on the device: the
    IEEE order keys of z through the in-house radix sort, then the middle
    element (odd n) or fl(fl(a + b) / 2) of the two middle ones (even n), as
    np.median computes it."""
    from .grid import radix_sort_pairs
    t = nat.torch()
    z, key, idx = _pose_depths_dev(field_.mu, pose, with_keys=True)
    n = int(z.numel())
    radix_sort_pairs(key, idx, 64)
    mid = idx[(n - 1) // 2:n // 2 + 1].to(t.int64)
    v = z[mid].cpu().numpy()
    return float(v[0]) if n % 2 else float((v[0] + v[1]) / 2)


def densify_and_prune(field_: GaussianField, window, cfg: SlamConfig, K: Optional[int] = None, *,
                      occupied=None, voxel_size: Optional[float] = None) -> GaussianField:
    """slam.py:601-651 — insert splats on the stride lattice of the newest
    keyframe, prune near-transparent ones, bump the generation.

    Reference semantics: lattice pixels whose rendered alpha (the GPU
    rasterizer, rasterizer.render) reaches ``coverage_alpha`` are skipped.
    Voxel variant (``occupied`` a :class:`grid.VoxelHashSet` and/or
    ``voxel_size`` given): lattice pixels whose voxel (default size the splat
    footprint max(min_scale, 0.5*stride*median_depth/fx)) is occupied by an
    existing centre are skipped instead of rendering coverage.
    """
    t = nat.require_cuda()
    if len(window) == 0:
        return field_
    kf = window.newest
    intr = frame_intrinsics(kf.frame, cfg)
    K = field_.K if K is None else K
    s = cfg.insert_stride
    median_depth = median_pose_depth(field_, kf.pose) if len(field_) else cfg.default_depth
    uu, vv = np.meshgrid(np.arange(0, intr.height, s), np.arange(0, intr.width, s), indexing="ij")
    uu, vv = uu.reshape(-1), vv.reshape(-1)
    if kf.frame.depth is not None:
        dsel = np.asarray(kf.frame.depth)[uu, vv]
        depth = np.where(dsel > 0, dsel.astype(np.float64), median_depth)
    else:
        depth = np.full(uu.size, median_depth)
    mu = backproject_pixels(kf.pose, intr, uu.astype(np.float64), vv.astype(np.float64), depth)
    if len(field_) and occupied is None and voxel_size is None:
        from .rasterizer import DEFAULT_RASTER, render
        alpha = render(field_, kf.pose, intr, cfg.raster if cfg.raster is not None else DEFAULT_RASTER).alpha
        alpha = alpha if isinstance(alpha, np.ndarray) else alpha.cpu().numpy()
        sel = ~(alpha[uu, vv] >= cfg.coverage_alpha)
        uu, vv, depth, mu = uu[sel], vv[sel], depth[sel], mu[sel]
    elif len(field_):
        from .grid import VoxelHashSet, pack_key
        vs = voxel_size if voxel_size is not None else max(cfg.min_scale, 0.5 * s * median_depth / intr.fx)
        occ = occupied
        if occ is None:
            occ = VoxelHashSet(2 * len(field_) + 1024)
            q = np.floor(field_.mu / vs).astype(np.int64)
            occ.insert(pack_key(q[:, 0], q[:, 1], q[:, 2]))
        q = np.floor(mu / vs).astype(np.int64)
        covered = occ.contains(pack_key(q[:, 0], q[:, 1], q[:, 2])).cpu().numpy()
        sel = ~covered
        uu, vv, depth, mu = uu[sel], vv[sel], depth[sel], mu[sel]
    size = np.maximum(cfg.min_scale, 0.5 * s * depth / intr.fx)
    color = np.asarray(kf.frame.color)[:, uu, vv].T
    n_new = uu.size
    keep = field_.opacity >= cfg.prune_opacity if len(field_) else np.zeros(0, bool)
    changed = (n_new > 0) or (len(field_) and not keep.all())
    if not changed:
        return field_

    def stack(old, extra):
        return np.concatenate([old[keep], extra]) if len(field_) else np.asarray(extra)

    return GaussianField(
        mu=stack(field_.mu, mu.reshape(n_new, 3)),
        quat=stack(field_.quat, np.tile([1.0, 0, 0, 0], (n_new, 1))),
        scale=stack(field_.scale, np.repeat(size[:, None], 3, axis=1).reshape(n_new, 3)),
        opacity=stack(field_.opacity, np.full(n_new, cfg.insert_opacity)),
        color=stack(field_.color, color.reshape(n_new, 3)),
        logits=stack(field_.logits, np.zeros((n_new, K))),
        generation=field_.generation + 1,
    )
