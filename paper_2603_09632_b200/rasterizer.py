"""Drop-in for ``semsplat.rasterizer`` (rasterizer.py:1-335) on the B200: the
lattice-only semantic rasterizer and its VJP.

``build_blend_pairs`` runs in libxgs as a tile-binned pipeline (csrc/raster.cu):
per-Gaussian projection + eigenvalue-floored screen covariance, an in-house
radix sort by depth, 16x16-pixel lattice tiles with depth-ordered splat lists,
and one CTA per tile compositing its lattice pixels front to back in fp64.
Channel accumulation (``render``, ``render_channels_grid``), the argmax ids
and the feature VJP reuse the pairs on the device; they only need the pairs
in front of each pixel's termination (dead pairs carry weight 0), so those
builds stop a tile once all of its pixels are terminated, while
``build_blend_pairs`` returns every culled pair as the reference does.  The codeword mixture
(decode) and the final softmax VJP go through ``core`` (libxgs + fp64 GEMM).

Fields are host ``GaussianField``s (copied to HBM per call) or any object
with CUDA-tensor ``mu``/``quat``/``scale``/``opacity``/``color``/``logits``;
outputs follow the field (NumPy for host fields, CUDA tensors otherwise).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import Codebook, decode_feature, device_f64, gemm_f64, is_tensor, softmax_vjp, to_host
from .errors import EmptySceneError, InvalidInputError
from .supervision import GridSpec

EIG_FLOOR_PX2 = 0.3


@dataclass(frozen=True)
class RasterConfig:
    """rasterizer.py:35-39."""

    term_threshold: float = 1e-4
    cutoff_sigma: float = 3.0
    eig_floor: float = EIG_FLOOR_PX2


DEFAULT_RASTER = RasterConfig()


@dataclass
class RenderOutput:
    color: object
    depth: object
    alpha: object
    blend_steps: int = 0


@dataclass
class CompactFeatureMap:
    data: object
    grid: GridSpec
    blend_steps: int = 0


@dataclass
class FeatureGradients:
    logit_grads: object
    feature_grads: object


@dataclass
class BlendPairs:
    gauss: object
    pixel: object
    weight: object
    alpha_prime: object
    t_before: object
    alive: object
    depth: object
    n_pixels: int
    blend_steps: int


def _step(a):
    a = np.asarray(a, dtype=np.int64).reshape(-1)
    if a.size == 0:
        return a, 0, 1
    s = int(a[1] - a[0]) if a.size > 1 else 1
    if s < 1 or np.any(a != a[0] + s * np.arange(a.size)):
        raise InvalidInputError("lattice rows/cols must be increasing arithmetic progressions")
    return a, int(a[0]), s


class _Pairs:
    """Device blend pairs of one (field, pose, lattice); freed on close/GC."""

    def __init__(self, field, pose, intr, rows, cols, cfg, all_pairs=False):
        t = nat.require_cuda()
        rows, r0, rs = _step(rows)
        cols, c0, cs = _step(cols)
        self.host = not is_tensor(field.mu)
        self.n = len(field)
        self.arrs = [device_f64(a) for a in (field.mu, field.quat, field.scale, field.opacity)]
        mu, quat, scale, opac = self.arrs
        ri = nat.RasterIn()
        ri.n = self.n
        ri.mu, ri.quat, ri.scale, ri.opacity = (a.data_ptr() for a in (mu, quat, scale, opac))
        R = np.asarray(pose.rotation, dtype=np.float64).reshape(9)
        tt = np.asarray(pose.translation, dtype=np.float64).reshape(3)
        for i in range(9):
            ri.R[i] = float(R[i])
        for i in range(3):
            ri.t[i] = float(tt[i])
        ri.fx, ri.fy, ri.cx, ri.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
        ri.near_z, ri.far_z = float(intr.near), float(intr.far)
        ri.n_rows, ri.row0, ri.row_step = rows.size, r0, rs
        ri.n_cols, ri.col0, ri.col_step = cols.size, c0, cs
        ri.term_threshold, ri.cutoff_sigma, ri.eig_floor = float(cfg.term_threshold), float(cfg.cutoff_sigma), \
            float(cfg.eig_floor)
        ri.all_pairs = 1 if all_pairs else 0
        self.shape = (rows.size, cols.size)
        self.n_pixels = rows.size * cols.size
        h = ctypes.c_void_p()
        npairs, steps = ctypes.c_int64(0), ctypes.c_int64(0)
        nat.call("xgs_raster_build", ctypes.byref(ri), ctypes.byref(h), ctypes.byref(npairs), ctypes.byref(steps),
                 nat.stream_ptr())
        self.h = h
        self.n_pairs, self.blend_steps = npairs.value, steps.value
        self.t = t

    def out(self, x):
        return to_host(x) if self.host else x

    def fetch(self) -> BlendPairs:
        t, m = self.t, self.n_pairs
        g = t.empty(m, dtype=t.int64, device="cuda")
        p = t.empty(m, dtype=t.int64, device="cuda")
        w, a, tb, d = (t.empty(m, dtype=t.float64, device="cuda") for _ in range(4))
        al = t.empty(m, dtype=t.uint8, device="cuda")
        nat.call("xgs_raster_fetch", self.h, nat.ptr(g), nat.ptr(p), nat.ptr(w), nat.ptr(a), nat.ptr(tb), nat.ptr(al),
                 nat.ptr(d), nat.stream_ptr())
        return BlendPairs(gauss=self.out(g), pixel=self.out(p), weight=self.out(w), alpha_prime=self.out(a),
                          t_before=self.out(tb), alive=self.out(al.bool()), depth=self.out(d),
                          n_pixels=self.n_pixels, blend_steps=self.blend_steps)

    def accumulate(self, payload, alpha=False, depth=False):
        t = self.t
        P = device_f64(payload, True) if payload is not None else None
        C = 0 if P is None else P.shape[1]
        out = t.empty((C, self.n_pixels), dtype=t.float64, device="cuda")
        a = t.empty(self.n_pixels, dtype=t.float64, device="cuda") if alpha else None
        d = t.empty(self.n_pixels, dtype=t.float64, device="cuda") if depth else None
        nat.call("xgs_raster_accumulate", self.h, nat.ptr(P), C, nat.ptr(out), nat.ptr(a), nat.ptr(d),
                 nat.stream_ptr())
        return out, a, d

    def argmax(self):
        o = self.t.empty(self.n_pixels, dtype=self.t.int64, device="cuda")
        nat.call("xgs_raster_argmax", self.h, nat.ptr(o), nat.stream_ptr())
        return o

    def vjp(self, upstream, D):
        t = self.t
        fg = t.empty((self.n, D), dtype=t.float64, device="cuda")
        nat.call("xgs_raster_vjp", self.h, nat.ptr(upstream), D, nat.ptr(fg), nat.stream_ptr())
        return fg

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            nat.lib().xgs_raster_free(self.h)
            self.h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_blend_pairs(field, pose, intr, rows, cols, cfg: RasterConfig = DEFAULT_RASTER) -> BlendPairs:
    """rasterizer.py:89-191 — depth-sorted, culled, terminated blend terms."""
    pr = _Pairs(field, pose, intr, rows, cols, cfg, all_pairs=True)
    try:
        return pr.fetch()
    finally:
        pr.close()


def _render(field, pose, intr, rows, cols, cfg):
    if len(field) == 0:
        raise EmptySceneError("cannot render an empty field")
    pr = _Pairs(field, pose, intr, rows, cols, cfg)
    try:
        col, a, d = pr.accumulate(field.color, alpha=True, depth=True)
        shape = pr.shape
        return RenderOutput(color=pr.out(col.reshape((3,) + shape)), depth=pr.out(d.reshape(shape)),
                            alpha=pr.out(a.reshape(shape)), blend_steps=pr.blend_steps)
    finally:
        pr.close()


def render(field, pose, intr, cfg: RasterConfig = DEFAULT_RASTER) -> RenderOutput:
    """rasterizer.py:215-229 — colour/depth/alpha at full resolution."""
    return _render(field, pose, intr, np.arange(intr.height), np.arange(intr.width), cfg)


def render_rect(field, pose, intr, rows, cols, cfg: RasterConfig = DEFAULT_RASTER) -> RenderOutput:
    """rasterizer.py:232-250 — the same per-pixel arithmetic on a row/column window."""
    return _render(field, pose, intr, rows, cols, cfg)


def render_channels_grid(field, payload, pose, intr, grid: GridSpec,
                         cfg: RasterConfig = DEFAULT_RASTER) -> CompactFeatureMap:
    """rasterizer.py:253-267 — composite a per-Gaussian payload (N, C) on the lattice."""
    if len(field) == 0:
        raise EmptySceneError("cannot render an empty field")
    if payload.shape[0] != len(field):
        raise InvalidInputError("payload rows must match Gaussian count")
    H_s, W_s = grid.H_s, grid.W_s
    host = not is_tensor(field.mu)
    if H_s == 0 or W_s == 0:
        z = np.zeros((payload.shape[1], H_s, W_s))
        return CompactFeatureMap(data=z if host else device_f64(z), grid=grid, blend_steps=0)
    pr = _Pairs(field, pose, intr, grid.rows(), grid.cols(), cfg)
    try:
        data, _, _ = pr.accumulate(payload)
        return CompactFeatureMap(data=pr.out(data.reshape(payload.shape[1], H_s, W_s)), grid=grid,
                                 blend_steps=pr.blend_steps)
    finally:
        pr.close()


def render_features_dense(field, codebook: Codebook, pose, intr, cfg: RasterConfig = DEFAULT_RASTER):
    """rasterizer.py:270-276 — dense (D, H, W) semantic feature map."""
    grid = GridSpec(H=intr.height, W=intr.width, s=1)
    return render_channels_grid(field, decode_feature(field.logits, codebook), pose, intr, grid, cfg).data


def render_features_grid(field, codebook: Codebook, pose, intr, grid: GridSpec,
                         cfg: RasterConfig = DEFAULT_RASTER) -> CompactFeatureMap:
    """rasterizer.py:279-284 — compact (D, H_s, W_s) features at the sampled pixels only."""
    return render_channels_grid(field, decode_feature(field.logits, codebook), pose, intr, grid, cfg)


def render_argmax_ids(field, pose, intr, cfg: RasterConfig = DEFAULT_RASTER):
    """rasterizer.py:287-306 — per-pixel Gaussian of the largest blend weight; -1 = none."""
    if len(field) == 0:
        raise EmptySceneError("cannot render an empty field")
    pr = _Pairs(field, pose, intr, np.arange(intr.height), np.arange(intr.width), cfg)
    try:
        return pr.out(pr.argmax().reshape(intr.height, intr.width))
    finally:
        pr.close()


def feature_gradients(field, codebook: Codebook, pose, intr, grid: GridSpec, upstream,
                      cfg: RasterConfig = DEFAULT_RASTER) -> FeatureGradients:
    """rasterizer.py:309-335 — backprop a (D, H_s, W_s) cotangent into per-Gaussian logits."""
    t = nat.require_cuda()
    host = not is_tensor(field.mu)
    up = device_f64(upstream)
    if tuple(up.shape) != (codebook.D, grid.H_s, grid.W_s):
        raise InvalidInputError(f"upstream shape {tuple(up.shape)} does not match (D, H_s, W_s)="
                                f"{(codebook.D, grid.H_s, grid.W_s)}")
    n = len(field)
    fg = t.zeros((n, codebook.D), dtype=t.float64, device="cuda")
    if grid.H_s and grid.W_s and n:
        pr = _Pairs(field, pose, intr, grid.rows(), grid.cols(), cfg)
        try:
            if pr.n_pairs:
                fg = pr.vjp(up.reshape(codebook.D, -1).contiguous(), codebook.D)
        finally:
            pr.close()
    E = codebook.E if codebook.on_device else device_f64(codebook.E, True)
    lg = softmax_vjp(device_f64(field.logits, True), gemm_f64(fg.contiguous(), E.contiguous(), b_transposed=True))
    return FeatureGradients(logit_grads=to_host(lg) if host else lg, feature_grads=to_host(fg) if host else fg)
