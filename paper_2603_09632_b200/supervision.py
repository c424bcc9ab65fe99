"""Drop-in for ``semsplat.supervision`` (supervision.py:1-221) on the B200.

Lattice bookkeeping (``GridSpec``, ``grid_resolution``, ``sample_coordinates``,
``next_offset``, ``padded_shape``) is host integer arithmetic exactly as in the
reference; the data-parallel parts -- target gathers and the masked semantic
loss -- run in libxgs (``xgs_sup_gather``, ``xgs_sup_loss``).
``prefetch_targets`` is the paper's "grid-sampled target prefetching"
(PAPER.md:246): the padded targets of a whole offset schedule in one launch.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as nat
from .core import is_tensor, to_host
from .errors import InvalidInputError, SemsplatError

NORM_EPS = 1e-8


class CorruptAnnotationError(SemsplatError, ValueError):
    """Region annotation references a region id outside its feature table (errors.py)."""


def grid_resolution(H: int, s: int, o: int) -> int:
    """supervision.py:21-31 (floored division; an offset past the last pixel -> 0)."""
    if s < 1:
        raise InvalidInputError("stride must be >= 1")
    if not (0 <= o < s):
        raise InvalidInputError("offset must satisfy 0 <= o < stride")
    return max(0, 1 + (H - 1 - o) // s)


@dataclass(frozen=True)
class GridSpec:
    """supervision.py:34-60."""

    H: int
    W: int
    s: int = 1
    o_h: int = 0
    o_w: int = 0

    def __post_init__(self):
        if self.s < 1:
            raise InvalidInputError("stride must be >= 1")
        if not (0 <= self.o_h < self.s and 0 <= self.o_w < self.s):
            raise InvalidInputError("offsets must satisfy 0 <= o < stride")

    @property
    def H_s(self) -> int:
        return grid_resolution(self.H, self.s, self.o_h)

    @property
    def W_s(self) -> int:
        return grid_resolution(self.W, self.s, self.o_w)

    def rows(self):
        return self.o_h + self.s * np.arange(self.H_s)

    def cols(self):
        return self.o_w + self.s * np.arange(self.W_s)


def sample_coordinates(grid: GridSpec):
    """supervision.py:63-67 — row-major (u, v) pairs."""
    uu, vv = np.meshgrid(grid.rows(), grid.cols(), indexing="ij")
    return np.stack([uu.ravel(), vv.ravel()], axis=1)


@dataclass
class SupervisionTarget:
    """supervision.py:70-81 (NumPy or CUDA tensors)."""

    G_star: object   # (D, H_s, W_s)
    V: object        # (1, H_s, W_s) binary


@dataclass
class RegionAnnotation:
    """supervision.py:84-97: region map S (-1 background) + R x D feature table."""

    S: object
    Phi: object

    @property
    def R(self) -> int:
        return int(self.Phi.shape[0])


@dataclass
class ContinuousFeatureSource:
    """supervision.py:100-115: P (D, H_f, W_f)."""

    P: object

    def __post_init__(self):
        if len(self.P.shape) != 3 or self.P.shape[1] < 1 or self.P.shape[2] < 1:
            raise InvalidInputError("feature source must be (D, H_f, W_f) with H_f, W_f >= 1")

    @property
    def H_f(self) -> int:
        return int(self.P.shape[1])

    @property
    def W_f(self) -> int:
        return int(self.P.shape[2])


def _dev(a, dtype):
    t = nat.torch()
    if is_tensor(a):
        return a.to(device="cuda", dtype=dtype).contiguous()
    np_dt = {t.float64: np.float64, t.float32: np.float32, t.int64: np.int64}[dtype]
    return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np_dt))).to("cuda")


def _gather(source, H, W, s, offsets, Hp, Wp):
    """Device targets for a list of offsets -> (G [n, D, Hp, Wp], V [n, 1, Hp, Wp])."""
    t = nat.require_cuda()
    offs = t.tensor(np.asarray(offsets, dtype=np.int32).reshape(-1, 2), device="cuda")
    n = int(offs.shape[0])
    corrupt = t.zeros(1, dtype=t.int32, device="cuda")
    if isinstance(source, ContinuousFeatureSource):
        P = source.P
        if not is_tensor(P) or P.dtype not in (t.float32, t.float64):
            P = _dev(P, t.float64)
        P = P.to("cuda").contiguous()
        D = int(P.shape[0])
        G = t.empty((n, D, Hp, Wp), dtype=t.float64, device="cuda")
        V = t.empty((n, 1, Hp, Wp), dtype=t.float64, device="cuda")
        nat.call("xgs_sup_gather", nat.ptr(P), nat.F32 if P.dtype == t.float32 else nat.F64, source.H_f,
                 source.W_f, None, None, 0, D, H, W, s, nat.ptr(offs), n, Hp, Wp, nat.ptr(G), nat.ptr(V),
                 nat.ptr(corrupt), nat.stream_ptr())
    else:
        S = _dev(source.S, t.int64)
        Phi = _dev(source.Phi, t.float64)
        if Phi.dim() < 2:
            Phi = Phi.reshape(1, -1)
        if tuple(S.shape) != (H, W):
            raise InvalidInputError("annotation resolution does not match grid")
        D = int(Phi.shape[1])
        G = t.empty((n, D, Hp, Wp), dtype=t.float64, device="cuda")
        V = t.empty((n, 1, Hp, Wp), dtype=t.float64, device="cuda")
        nat.call("xgs_sup_gather", None, nat.F64, 0, 0, nat.ptr(S), nat.ptr(Phi), int(Phi.shape[0]), D, H, W, s,
                 nat.ptr(offs), n, Hp, Wp, nat.ptr(G), nat.ptr(V), nat.ptr(corrupt), nat.stream_ptr())
        if int(corrupt.item()):
            raise CorruptAnnotationError("region index outside feature table")
    return G, V


def _host_mode(*objs):
    return not any(is_tensor(o) for o in objs)


def build_target_discrete(ann: RegionAnnotation, grid: GridSpec) -> SupervisionTarget:
    """supervision.py:118-130 — table lookup, background (-1) masked."""
    G, V = _gather(ann, grid.H, grid.W, grid.s, [(grid.o_h, grid.o_w)], grid.H_s, grid.W_s)
    if _host_mode(ann.S, ann.Phi):
        return SupervisionTarget(G_star=to_host(G[0]), V=to_host(V[0]))
    return SupervisionTarget(G_star=G[0], V=V[0])


def build_target_continuous(src: ContinuousFeatureSource, grid: GridSpec) -> SupervisionTarget:
    """supervision.py:138-147 — nearest-neighbour alignment onto the feature map."""
    G, V = _gather(src, grid.H, grid.W, grid.s, [(grid.o_h, grid.o_w)], grid.H_s, grid.W_s)
    if _host_mode(src.P):
        return SupervisionTarget(G_star=to_host(G[0]), V=to_host(V[0]))
    return SupervisionTarget(G_star=G[0], V=V[0])


def masked_semantic_loss(pred, target: SupervisionTarget, lambda_sem: float = 1.0):
    """supervision.py:150-184 — masked cosine + L1 loss and its cotangent."""
    t = nat.require_cuda()
    host = _host_mode(pred, target.G_star)
    P = _dev(pred, t.float64)
    G = _dev(target.G_star, t.float64)
    V = _dev(target.V, t.float64)
    if tuple(P.shape) != tuple(G.shape):
        raise InvalidInputError("prediction and target shapes disagree")
    D = int(P.shape[0])
    cells = int(P[0].numel())
    acc = t.zeros(3, dtype=t.float64, device="cuda")
    cot = t.empty_like(P)
    nat.call("xgs_sup_loss", nat.ptr(P), nat.ptr(G), nat.ptr(V), D, cells, float(lambda_sem), nat.ptr(acc),
             nat.ptr(cot), nat.stream_ptr())
    s_cos, s_l1, n = (float(v) for v in acc.cpu())
    loss = 0.0 if n == 0 else lambda_sem * (s_cos / n + s_l1 / n)
    return float(loss), (to_host(cot) if host else cot)


def next_offset(step: int, s: int, rng_seed: int = 0):
    """supervision.py:187-202 — seeded permutation of the s^2 phases, cyclic."""
    if s < 1:
        raise InvalidInputError("stride must be >= 1")
    if s == 1:
        return (0, 0)
    n = s * s
    cycle, pos = divmod(int(step), n)
    perm = np.random.default_rng([int(rng_seed), cycle]).permutation(n)
    k = int(perm[pos])
    return (k // s, k % s)


def padded_shape(H: int, W: int, s: int):
    """supervision.py:204-206."""
    return (-(-H // s), -(-W // s))


def pad_target(target: SupervisionTarget, grid: GridSpec) -> SupervisionTarget:
    """supervision.py:208-221 — pad to the offset-independent batched shape."""
    t = nat.require_cuda()
    host = _host_mode(target.G_star)
    Hp, Wp = padded_shape(grid.H, grid.W, grid.s)
    G = _dev(target.G_star, t.float64)
    V = _dev(target.V, t.float64)
    Gp = t.zeros((G.shape[0], Hp, Wp), dtype=t.float64, device="cuda")
    Vp = t.zeros((1, Hp, Wp), dtype=t.float64, device="cuda")
    Gp[:, :grid.H_s, :grid.W_s] = G
    Vp[:, :grid.H_s, :grid.W_s] = V
    return SupervisionTarget(G_star=to_host(Gp) if host else Gp, V=to_host(Vp) if host else Vp)


def prefetch_targets(source, H: int, W: int, s: int, steps: Sequence[int], rng_seed: int = 0):
    """Padded targets for the offsets of ``steps`` (``next_offset`` schedule) in
    one launch: (G [n, D, Hp, Wp], V [n, 1, Hp, Wp]) CUDA tensors, equal to
    ``pad_target(build_target_*(source, GridSpec(H, W, s, *next_offset(k, s, seed))))``."""
    offs = [next_offset(k, s, rng_seed) for k in steps]
    Hp, Wp = padded_shape(H, W, s)
    return _gather(source, H, W, s, offs, Hp, Wp)
