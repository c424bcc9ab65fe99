"""State types of the hot path, mirroring semsplat.core (core.py:1-315).

Conventions (core.py:1-10): CameraPose is world->camera, x_cam = R x_w + t;
image coordinates (u, v) = (row, column), row u pairs with fx/cx and column v
with fy/cy.

``Codebook`` / ``FeatureReservoir`` accept NumPy arrays (the reference's
types, copied to the B200 per call) or CUDA tensors (device-resident; results
stay on the device).  The reservoir is a device ring buffer in both cases.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .errors import InvalidInputError

QUAT_NORM_TOL = 1e-6


def is_tensor(a):
    if nat._torch is None and type(a).__module__.split(".")[0] != "torch":
        return False
    return isinstance(a, nat.torch().Tensor)


def device_f64(a, shape_2d=False):
    """NumPy / torch -> contiguous fp64 CUDA tensor."""
    t = nat.require_cuda()
    if is_tensor(a):
        out = a.to(device="cuda", dtype=t.float64)
    else:
        out = t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).to("cuda")
    if shape_2d and out.dim() < 2:
        out = out.reshape(1, -1)
    return out.contiguous()


def to_host(t):
    return t.detach().cpu().numpy()


class FeatureReservoir:
    """Bounded FIFO of the most recent feature rows (core.py:178-203), kept as
    an fp64 ring buffer in HBM; ``extend`` copies only the last ``capacity``
    rows of a batch."""

    def __init__(self, capacity: int, dim: int):
        if capacity < 1:
            raise InvalidInputError("reservoir capacity must be >= 1")
        self.capacity = int(capacity)
        self.dim = int(dim)
        self._ring = None
        self._head = 0
        self._len = 0

    def __len__(self) -> int:
        return self._len

    def _ensure(self):
        if self._ring is None:
            t = nat.require_cuda()
            self._ring = t.empty((self.capacity, self.dim), dtype=t.float64, device="cuda")
        return self._ring

    def _extend_rows(self, xt, dtype, n, ldx):
        """Append rows of a CUDA row-major buffer (FIFO keeps the last cap)."""
        ring = self._ensure()
        cap = self.capacity
        if n == 0:
            return
        if n >= cap:
            nat.call("xgs_vq_ring_write", nat.ptr(xt), dtype, ldx, n - cap, cap, self.dim, nat.ptr(ring),
                     cap, 0, nat.stream_ptr())
            self._head, self._len = 0, cap
            return
        start = (self._head + self._len) % cap
        nat.call("xgs_vq_ring_write", nat.ptr(xt), dtype, ldx, 0, n, self.dim, nat.ptr(ring), cap, start,
                 nat.stream_ptr())
        self._account(n)

    def _account(self, n):
        """FIFO bookkeeping of an append of n rows (the rows themselves written
        by the caller, e.g. xgs_vq_ring_write_dev inside a CUDA graph)."""
        cap = self.capacity
        if n <= 0:
            return
        if n >= cap:
            self._head, self._len = 0, cap
            return
        total = self._len + n
        if total > cap:
            self._head = (self._head + total - cap) % cap
            self._len = cap
        else:
            self._len = total

    def _write_pos(self):
        """Physical ring row of the next append."""
        return (self._head + self._len) % self.capacity

    def extend(self, x) -> None:
        from .vq import _rows
        xt, dtype, n, d, ldx = _rows(x)
        if d != self.dim:
            raise InvalidInputError("reservoir dimension mismatch")
        self._extend_rows(xt, dtype, n, ldx)

    def _draw(self, rng) -> int:
        """One reference draw (core.py:199): physical ring row of rng.integers(0, len)."""
        i = int(rng.integers(0, len(self)))
        return (self._head + i) % self.capacity

    def sample(self, rng) -> np.ndarray:
        if len(self) == 0:
            raise InvalidInputError("cannot sample from an empty reservoir")
        return to_host(self._ring[self._draw(rng)])

    def as_array(self) -> np.ndarray:
        if self._len == 0:
            return np.empty((0, self.dim))
        idx = [(self._head + i) % self.capacity for i in range(self._len)]
        return to_host(self._ring[idx])


@dataclass
class Codebook:
    """K x D codewords plus EMA count/sum buffers and a reservoir (core.py:206-243)."""

    E: object
    N: object
    M: object
    lam: float
    epsilon: float
    reservoir: FeatureReservoir = field(repr=False, default=None)

    def __post_init__(self):
        if is_tensor(self.E) or is_tensor(self.N) or is_tensor(self.M):
            self.E = device_f64(self.E, shape_2d=True)
            self.N = device_f64(self.N).reshape(-1)
            self.M = device_f64(self.M, shape_2d=True)
            neg = bool((self.N < 0).any()) if self.N.numel() else False
        else:
            self.E = np.atleast_2d(np.asarray(self.E, dtype=np.float64))
            self.N = np.asarray(self.N, dtype=np.float64).reshape(-1)
            self.M = np.atleast_2d(np.asarray(self.M, dtype=np.float64))
            neg = bool(np.any(self.N < 0))
        if tuple(self.E.shape) != tuple(self.M.shape) or self.N.shape[0] != self.E.shape[0]:
            raise InvalidInputError("codebook buffer shapes disagree")
        if not (0.0 <= self.lam < 1.0):
            raise InvalidInputError("EMA decay must lie in [0, 1)")
        if neg:
            raise InvalidInputError("EMA counts must be nonnegative")
        if self.reservoir is None:
            self.reservoir = FeatureReservoir(4096, self.E.shape[1])

    @classmethod
    def _make(cls, E, N, M, lam, epsilon, reservoir):
        """Trusted constructor for kernel outputs (no host sync for validation:
        N >= 0 holds by construction of the EMA / revival updates)."""
        cb = object.__new__(cls)
        cb.E, cb.N, cb.M = E, N, M
        cb.lam, cb.epsilon, cb.reservoir = lam, epsilon, reservoir
        return cb

    @property
    def K(self) -> int:
        return int(self.E.shape[0])

    @property
    def D(self) -> int:
        return int(self.E.shape[1])

    @property
    def on_device(self) -> bool:
        return is_tensor(self.E)

    @staticmethod
    def zeros(K: int, D: int, lam: float = 0.96, epsilon: float = 1e-5,
              reservoir_capacity: int = 4096) -> "Codebook":
        return Codebook(E=np.zeros((K, D)), N=np.zeros(K), M=np.zeros((K, D)), lam=lam, epsilon=epsilon,
                        reservoir=FeatureReservoir(reservoir_capacity, D))

    def to_device(self) -> "Codebook":
        return Codebook._make(device_f64(self.E, True), device_f64(self.N).reshape(-1),
                              device_f64(self.M, True), self.lam, self.epsilon, self.reservoir)

    def to_numpy(self) -> "Codebook":
        if not self.on_device:
            return self
        return Codebook._make(to_host(self.E), to_host(self.N), to_host(self.M), self.lam, self.epsilon,
                              self.reservoir)


@dataclass
class CameraPose:
    """World-to-camera rigid transform (core.py:246-295)."""

    rotation: np.ndarray
    translation: np.ndarray

    def __post_init__(self):
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        if np.max(np.abs(self.rotation @ self.rotation.T - np.eye(3))) > 1e-6:
            raise InvalidInputError("pose rotation must be orthonormal within 1e-6")
        if abs(np.linalg.det(self.rotation) - 1.0) > 1e-6:
            raise InvalidInputError("pose rotation must have det +1")

    @staticmethod
    def identity() -> "CameraPose":
        return CameraPose(np.eye(3), np.zeros(3))

    def transform(self, pts):
        pts = np.asarray(pts, dtype=np.float64)
        return pts @ self.rotation.T + self.translation

    def camera_center(self):
        return -self.rotation.T @ self.translation


@dataclass
class CameraIntrinsics:
    """Pinhole intrinsics (core.py:298-315); u = row <-> fx/cx."""

    fx: float
    fy: float
    cx: float
    cy: float
    height: int
    width: int
    near: float = 0.05
    far: float = 100.0

    def __post_init__(self):
        if self.fx <= 0 or self.fy <= 0:
            raise InvalidInputError("focal lengths must be positive")
        if not (0 < self.near < self.far):
            raise InvalidInputError("require 0 < near < far")

    @staticmethod
    def from_fov(height: int, width: int, fov_deg: float = 60.0, near: float = 0.05,
                 far: float = 100.0) -> "CameraIntrinsics":
        f = 0.5 * min(height, width) / np.tan(np.deg2rad(fov_deg) / 2)
        return CameraIntrinsics(fx=f, fy=f, cx=(height - 1) / 2, cy=(width - 1) / 2, height=height,
                                width=width, near=near, far=far)


@dataclass
class GaussianField:
    """Struct-of-arrays Gaussian map (core.py:107-175)."""

    mu: np.ndarray
    quat: np.ndarray
    scale: np.ndarray
    opacity: np.ndarray
    color: np.ndarray
    logits: np.ndarray
    generation: int = 0

    def __post_init__(self):
        self.mu = np.atleast_2d(np.asarray(self.mu, dtype=np.float64))
        self.quat = np.atleast_2d(np.asarray(self.quat, dtype=np.float64))
        self.scale = np.atleast_2d(np.asarray(self.scale, dtype=np.float64))
        self.opacity = np.asarray(self.opacity, dtype=np.float64).reshape(-1)
        self.color = np.atleast_2d(np.asarray(self.color, dtype=np.float64))
        self.logits = np.atleast_2d(np.asarray(self.logits, dtype=np.float64))
        n = self.mu.shape[0]
        if not (self.quat.shape == (n, 4) and self.scale.shape == (n, 3) and self.opacity.shape == (n,)
                and self.color.shape == (n, 3) and self.logits.shape[0] == n):
            raise InvalidInputError("inconsistent field array shapes")
        norms = np.linalg.norm(self.quat, axis=1)
        if n and np.max(np.abs(norms - 1.0)) > QUAT_NORM_TOL:
            raise InvalidInputError("field quaternions must be unit-norm within 1e-6")
        if n and np.any(self.scale <= 0):
            raise InvalidInputError("field scales must be strictly positive")
        self.opacity = np.clip(self.opacity, 0.0, 1.0)

    def __len__(self) -> int:
        return self.mu.shape[0]

    @property
    def K(self) -> int:
        return self.logits.shape[1]


# ------------------------------------------------------------ codebook consumers
# core.py:473-496 of the reference.  NumPy in -> NumPy out (one H2D/D2H copy per
# call); CUDA tensors in -> CUDA tensors out.  The row ops run in libxgs
# (xgs_softmax_rows: fp64, NumPy's max / exp / pairwise-sum order); the
# codeword mixture softmax(logits) @ E is xgs_gemm_f64 (softmax fused into the
# fp64 DMMA contraction).

SOFTMAX_WEIGHTS, SOFTMAX_ENTROPY, SOFTMAX_VJP = 1, 2, 4


def _logits_dev(logits):
    host = not is_tensor(logits)
    t = nat.require_cuda()
    L = device_f64(logits)
    squeeze = L.dim() == 1
    if squeeze:
        L = L.reshape(1, -1)
    if L.dim() != 2:
        raise InvalidInputError("logits must be (K,) or (N, K)")
    return t, L.contiguous(), host, squeeze


def _softmax_rows(L, mode, upstream=None):
    t = nat.torch()
    n, k = L.shape
    out = t.empty((n, k), dtype=t.float64, device="cuda") if mode != SOFTMAX_ENTROPY else None
    out_h = t.empty(n, dtype=t.float64, device="cuda") if mode == SOFTMAX_ENTROPY else None
    nat.call("xgs_softmax_rows", nat.ptr(L), n, k, mode, nat.ptr(upstream), nat.ptr(out), nat.ptr(out_h),
             nat.stream_ptr())
    return out if mode != SOFTMAX_ENTROPY else out_h


def _ret(x, host, squeeze):
    if squeeze:
        x = x[0]
    return to_host(x) if host else x


def mixture_weights(logits):
    """core.py:473-480 — stable softmax over the codeword axis."""
    t, L, host, squeeze = _logits_dev(logits)
    return _ret(_softmax_rows(L, SOFTMAX_WEIGHTS), host, squeeze)


def softmax_vjp(logits, upstream):
    """core.py:483-487 — w * (upstream - sum(w * upstream))."""
    t, L, host, squeeze = _logits_dev(logits)
    U = device_f64(upstream).reshape(L.shape).contiguous()
    return _ret(_softmax_rows(L, SOFTMAX_VJP, U), host, squeeze)


def gemm_f64(A, B, softmax=False, b_transposed=False, a_transposed=False, query=None, tau=1.0, eps=0.0,
             want_c=True):
    """xgs_gemm_f64 (fp64 DMMA contraction, csrc/decode_f64.cu) on CUDA fp64
    tensors: C = op(A) . B where op(A) = softmax over A's rows when `softmax`;
    A is (n, kr) (or (kr, n) read transposed), B is (kr, m) (or (m, kr) read
    transposed).  With `query` (nq, m) also / instead returns the contrast
    scores of thinker.py:110-129 per row (no C needed)."""
    t = nat.torch()
    n, kr = (A.shape[1], A.shape[0]) if a_transposed else (A.shape[0], A.shape[1])
    m = B.shape[0] if b_transposed else B.shape[1]
    if (B.shape[1] if b_transposed else B.shape[0]) != kr:
        raise InvalidInputError("inner dimensions disagree")
    lda_r, lda_k = (A.stride(1), A.stride(0)) if a_transposed else (A.stride(0), A.stride(1))
    ldb_k, ldb_m = (B.stride(1), B.stride(0)) if b_transposed else (B.stride(0), B.stride(1))
    C = t.empty((n, m), dtype=t.float64, device="cuda") if want_c else None
    scores = t.empty(n, dtype=t.float64, device="cuda") if query is not None else None
    nq = int(query.shape[0]) if query is not None else 0
    if softmax and a_transposed:
        A = A.t().contiguous()
        lda_r, lda_k = A.stride(0), A.stride(1)
    ws = nat.workspace("gemm_f64", nat.lib().xgs_gemm_f64_workspace(n, kr, m, nq, 1 if softmax else 0))
    nat.call("xgs_gemm_f64", nat.ptr(A), n, kr, lda_r, lda_k, 1 if softmax else 0, nat.ptr(B), m, ldb_k, ldb_m,
             nat.ptr(C), m, nat.ptr(query), nq, float(tau), float(eps), nat.ptr(scores), nat.ptr(ws), ws.numel(),
             nat.stream_ptr())
    return C if query is None else (C, scores)


def decode_feature(logits, codebook: "Codebook"):
    """core.py:490-496 — softmax-weighted codeword mixture, (K,) or (N, K) logits:
    softmax and contraction fused in one fp64 DMMA kernel (xgs_gemm_f64)."""
    t, L, host, squeeze = _logits_dev(logits)
    if L.shape[-1] != codebook.K:
        raise InvalidInputError(f"logit length {L.shape[-1]} does not match codebook K={codebook.K}")
    if not bool(t.isfinite(L).all()):
        raise InvalidInputError("logits must be finite")
    E = codebook.E if codebook.on_device else device_f64(codebook.E, True)
    return _ret(gemm_f64(L, E.contiguous(), softmax=True), host, squeeze)
