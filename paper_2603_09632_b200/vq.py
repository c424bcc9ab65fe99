"""Drop-in replacement for ``semsplat.vq`` (vq.py:1-230) running on the B200.

Same names, signatures, return types and error behaviour as the reference:
NumPy in -> NumPy out (the arrays are copied to HBM per call), CUDA tensors in
-> CUDA tensors out with no host round trip except the tiny dead-code
readback that the reference's host RNG needs.  Every distance, argmin,
count/sum, EMA and revival is computed by libxgs kernels; results are
bit-identical to the reference on one GPU (codes, counts, sums, E, N, M).

Hot path (``online_step``, vq.py:193-212):
  reservoir ring write -> [confidence mask] -> tcgen05 screening GEMM +
  exact re-rank (codes) -> counting-sort + sequential fp64 chains (stats) ->
  EMA kernel -> host RNG draws -> revival kernel.
"""

from __future__ import annotations

import csv
import ctypes
import threading
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _native as nat
from .core import Codebook, FeatureReservoir, is_tensor, to_host, device_f64
from .errors import InvalidInputError, InvalidStateError


@dataclass
class VqConfig:
    """vq.py:21-39 (same defaults and validation)."""

    K: int = 256
    lam: float = 0.96
    tau_warm: float = 0.7
    gamma: float = 0.5
    delta_dead: float = 1e-2
    epsilon: float = 1e-5
    reservoir_capacity: int = 4096

    def __post_init__(self):
        if not (0.0 <= self.lam < 1.0):
            raise InvalidInputError("lam must lie in [0, 1)")
        if self.K < 1:
            raise InvalidInputError("K must be >= 1")
        if not (0.0 < self.gamma < 1.0):
            raise InvalidInputError("gamma must lie in (0, 1)")
        if self.delta_dead <= 0:
            raise InvalidInputError("delta_dead must be positive")


@dataclass
class VqBatchStats:
    counts: object  # (K,) integer-valued fp64
    sums: object    # (K, D) fp64


@dataclass
class WarmStartResult:
    codebook: Codebook
    used: int
    degenerate: bool


@dataclass
class ReviveResult:
    codebook: Codebook
    revived: list
    skipped: bool


# ---------------------------------------------------------------- plumbing

def _rows(x):
    """Any row batch -> (CUDA tensor, dtype code, n, d, ldx); mirrors the
    reference's atleast_2d + fp64 cast (vq.py:62-66) without widening on the
    host: fp32 / bf16 / fp64 go to the device as-is (widening is exact)."""
    t = nat.require_cuda()
    if is_tensor(x):
        xt = x
        if xt.dim() < 2:
            xt = xt.reshape(1, -1)
        if xt.dim() != 2:
            raise InvalidInputError("feature batch must be 1-D or 2-D")
        if xt.dtype not in (t.float32, t.float64, t.bfloat16):
            xt = xt.to(t.float64)
        if xt.device.type != "cuda":
            xt = xt.to("cuda")
    else:
        a = np.asarray(x)
        if a.dtype not in (np.float32, np.float64):
            a = a.astype(np.float64)
        a = np.atleast_2d(a)
        if a.ndim != 2:
            raise InvalidInputError("feature batch must be 1-D or 2-D")
        xt = t.from_numpy(np.ascontiguousarray(a)).to("cuda")
    n, d = int(xt.shape[0]), int(xt.shape[1])
    if n > 0 and (xt.stride(1) != 1 or (n > 1 and xt.stride(0) < d)):
        xt = xt.contiguous()
    ldx = int(xt.stride(0)) if n > 1 else d
    ldx = max(ldx, d)
    return xt, nat.dtype_code(xt), n, d, ldx


def _host_mode(*objs):
    """Reference types in -> reference types out."""
    for o in objs:
        if isinstance(o, Codebook):
            if o.on_device:
                return False
        elif is_tensor(o):
            return False
    return True


def _out(t, host):
    return to_host(t) if host else t


def _check_d(d, codebook):
    if d != codebook.D:
        raise InvalidInputError(f"feature dim {d} != codebook D={codebook.D}")


def _E(codebook):
    return codebook.E if codebook.on_device else device_f64(codebook.E, True)


def _assign_dev(xt, dt, n, d, ldx, E, K, stats=False):
    t = nat.torch()
    codes = t.empty(n, dtype=t.int64, device="cuda")
    if n == 0:
        return (codes, (0, 0)) if stats else codes
    ws = nat.workspace("assign", nat.lib().xgs_vq_assign_workspace(n, K, d, dt, ldx))
    st = (ctypes.c_int32 * 2)() if stats else None
    nat.call("xgs_vq_assign", nat.ptr(xt), dt, n, d, ldx, nat.ptr(E), K, nat.ptr(codes), nat.ptr(ws),
             ws.numel(), st, nat.stream_ptr())
    return (codes, (st[0], st[1])) if stats else codes


def _exact_dev(xt, dt, n, d, ldx, E, K, mode, tau=1.0, gamma=0.5):
    t = nat.torch()
    dist = t.empty((n, K), dtype=t.float64, device="cuda") if mode & nat.EX_DIST else None
    prob = t.empty((n, K), dtype=t.float64, device="cuda") if mode & nat.EX_PROB else None
    codes = t.empty(n, dtype=t.int64, device="cuda") if mode & nat.EX_CODE else None
    mask = t.empty(n, dtype=t.uint8, device="cuda") if mode & nat.EX_MASK else None
    if n:
        nat.call("xgs_vq_exact", nat.ptr(xt), dt, n, d, ldx, nat.ptr(E), K, mode, float(tau), float(gamma),
                 nat.ptr(dist), nat.ptr(prob), nat.ptr(codes), nat.ptr(mask), nat.stream_ptr())
        if mask is not None:
            _decide_borderline(xt, dt, n, d, ldx, E, K, mask, tau, gamma)
    return dist, prob, codes, mask


def _decide_borderline(xt, dt, n, d, ldx, E, K, mask, tau, gamma):
    """Rows the kernel marked 2 (fl(1/S) within 1e-12 relative of gamma,
    where a last-ulp difference between CUDA's exp and the host libm's could
    flip the decision) are decided with the reference's own NumPy expression
    (vq.py:112-124) on their exact fp64 distances (bit-identical to
    squared_distances)."""
    t = nat.torch()
    idx = (mask == 2).nonzero().reshape(-1)
    if idx.numel() == 0:
        return
    sub = xt[:n].index_select(0, idx).contiguous()
    dist, _, _, _ = _exact_dev(sub, dt, int(idx.numel()), d, d, E, K, nat.EX_DIST)
    sq = dist.cpu().numpy()
    dd = np.sqrt(sq)
    logits = -dd / tau
    logits -= logits.max(axis=1, keepdims=True)
    e = np.exp(logits)
    p = e / e.sum(axis=1, keepdims=True)
    ok = p.max(axis=1) >= gamma
    mask[idx] = t.from_numpy(ok.astype(np.uint8)).to(mask.device)


def _accumulate_dev(xt, dt, n, d, ldx, codes, mask, K):
    t = nat.torch()
    counts = t.empty(K, dtype=t.float64, device="cuda")
    sums = t.empty((K, d), dtype=t.float64, device="cuda")
    ws = nat.workspace("accumulate", nat.lib().xgs_vq_accumulate_workspace(n, K))
    nat.call("xgs_vq_accumulate", nat.ptr(xt), dt, n, d, ldx, nat.ptr(codes), nat.ptr(mask), K,
             nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel(), nat.stream_ptr())
    return counts, sums


_STEP_WS = {}


def _step_ws_bytes(n, K, d, dt, ldx):
    """xgs_vq_step_workspace, memoised (a pure function of the shape; called every step)."""
    key = (n, K, d, dt, ldx)
    b = _STEP_WS.get(key)
    if b is None:
        if len(_STEP_WS) > 64:
            _STEP_WS.clear()
        b = _STEP_WS[key] = int(nat.lib().xgs_vq_step_workspace(n, K, d, dt, ldx))
    return b


def _assign_accumulate_dev(xt, dt, n, d, ldx, E, K, counts=None, sums=None, x_host=None):
    """assign_batch + accumulate(batch) for an all-pass mask (vq.py:206) in one
    row-chunk-pipelined native call; bit-identical to _assign_dev followed by
    _accumulate_dev.  ``x_host`` (pinned CPU tensor, same layout as ``xt``):
    the rows are streamed into ``xt`` chunk by chunk inside the call."""
    t = nat.torch()
    codes = t.empty(n, dtype=t.int64, device="cuda")
    if counts is None:
        counts = t.empty(K, dtype=t.float64, device="cuda")
    if sums is None:
        sums = t.empty((K, d), dtype=t.float64, device="cuda")
    ws = nat.workspace("step", _step_ws_bytes(n, K, d, dt, ldx))
    nat.call("xgs_vq_assign_accumulate_h2d", nat.ptr(x_host), nat.ptr(xt), dt, n, d, ldx, nat.ptr(E), K,
             nat.ptr(codes), nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel(), None, nat.stream_ptr())
    return codes, counts, sums


def _ema_dev(codebook, counts, sums):
    t = nat.torch()
    N = device_f64(codebook.N).reshape(-1) if not codebook.on_device else codebook.N
    M = device_f64(codebook.M, True) if not codebook.on_device else codebook.M
    K, D = codebook.K, codebook.D
    N2 = t.empty_like(N)
    M2 = t.empty_like(M)
    E2 = t.empty_like(M)
    nat.call("xgs_vq_ema", float(codebook.lam), float(codebook.epsilon), K, D, nat.ptr(N), nat.ptr(M),
             nat.ptr(counts), nat.ptr(sums), nat.ptr(N2), nat.ptr(M2), nat.ptr(E2), nat.stream_ptr())
    return E2, N2, M2


def all_pass_provable(gamma: float, K: int) -> bool:
    """max softmax >= 1/K always (vq.py:112-124), so gamma below 1/K (with a
    margin for libm ulps) makes the confidence mask all-true."""
    return gamma <= (1.0 / K) * (1.0 - 1e-9)


# ---------------------------------------------------------------- public API

def squared_distances(x, codebook: Codebook):
    """vq.py:69-73 — exact fp64 (N, K), NumPy pairwise summation order."""
    xt, dt, n, d, ldx = _rows(x)
    _check_d(d, codebook)
    dist, _, _, _ = _exact_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K, nat.EX_DIST)
    return _out(dist, _host_mode(x, codebook))


def assign(x, codebook: Codebook) -> int:
    """vq.py:76-81 — nearest codeword of one sample, lowest index on ties."""
    if codebook.K == 0:
        raise InvalidStateError("cannot assign against an empty codebook")
    if not is_tensor(x):
        x = np.asarray(x, dtype=np.float64)[None]
    xt, dt, n, d, ldx = _rows(x)
    _check_d(d, codebook)
    return int(_assign_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K)[0].item())


def assign_batch(x, codebook: Codebook):
    """vq.py:84-87 — int64 codes (tcgen05 screen + exact fp64 re-rank)."""
    if codebook.K == 0:
        raise InvalidStateError("cannot assign against an empty codebook")
    xt, dt, n, d, ldx = _rows(x)
    _check_d(d, codebook)
    return _out(_assign_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K), _host_mode(x, codebook))


def assign_batch_stats(x, codebook: Codebook):
    """assign_batch plus (rows re-ranked exactly, rows rescanned over all K)."""
    xt, dt, n, d, ldx = _rows(x)
    _check_d(d, codebook)
    codes, st = _assign_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K, stats=True)
    return _out(codes, _host_mode(x, codebook)), st


def accumulate(batch, codebook: Codebook) -> VqBatchStats:
    """vq.py:90-100 — per-code counts and sums, bit-identical to np.add.at."""
    xt, dt, n, d, ldx = _rows(batch)
    _check_d(d, codebook)
    if n == 0:
        raise InvalidInputError("batch must be nonempty")
    if codebook.K == 0:
        raise InvalidStateError("cannot assign against an empty codebook")
    codes = _assign_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K)
    counts, sums = _accumulate_dev(xt, dt, n, d, ldx, codes, None, codebook.K)
    host = _host_mode(batch, codebook)
    return VqBatchStats(counts=_out(counts, host), sums=_out(sums, host))


def ema_step(codebook: Codebook, stats: VqBatchStats) -> Codebook:
    """vq.py:103-109 — decay toward the batch statistics (lam from the codebook)."""
    host = _host_mode(codebook, stats.counts, stats.sums)
    counts = device_f64(stats.counts).reshape(-1)
    sums = device_f64(stats.sums, True)
    if counts.shape[0] != codebook.K or tuple(sums.shape) != (codebook.K, codebook.D):
        raise InvalidInputError("batch statistics do not match the codebook")
    E, N, M = _ema_dev(codebook, counts, sums)
    if host:
        return Codebook(E=to_host(E), N=to_host(N), M=to_host(M), lam=codebook.lam, epsilon=codebook.epsilon,
                        reservoir=codebook.reservoir)
    return Codebook._make(E, N, M, codebook.lam, codebook.epsilon, codebook.reservoir)


def confidence_scores(batch, codebook: Codebook, tau: float):
    """vq.py:112-118 — softmax over -sqrt(d)/tau (exact fp64 distances)."""
    xt, dt, n, d, ldx = _rows(batch)
    _check_d(d, codebook)
    _, prob, _, _ = _exact_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K, nat.EX_PROB, tau=tau)
    return _out(prob, _host_mode(batch, codebook))


def confidence_mask(batch, codebook: Codebook, cfg: VqConfig):
    """vq.py:121-124 — rows whose max confidence reaches gamma."""
    xt, dt, n, d, ldx = _rows(batch)
    _check_d(d, codebook)
    host = _host_mode(batch, codebook)
    if all_pass_provable(cfg.gamma, codebook.K):
        t = nat.torch()
        m = t.ones(n, dtype=t.bool, device="cuda")
    else:
        _, _, _, m = _exact_dev(xt, dt, n, d, ldx, _E(codebook), codebook.K, nat.EX_MASK, tau=cfg.tau_warm,
                                gamma=cfg.gamma)
        m = m.bool()
    return _out(m, host)


def seed_from_samples(buffer, K: int):
    """vq.py:126-147 — greedy farthest-point seeding.  The K-1 argmax passes run
    as back-to-back launches of xgs_vq_seed_farthest (seed indices stay on the
    device; no host round trip per seed)."""
    t = nat.require_cuda()
    host = _host_mode(buffer)
    xt, dt, n, d, ldx = _rows(buffer)
    if n == 0:
        raise InvalidInputError("seed buffer must be nonempty")
    K = max(int(K), 1)   # the reference always returns at least buffer[0]
    seeds = t.empty(K, dtype=t.int64, device="cuda")
    ws = nat.workspace("seed", nat.lib().xgs_vq_seed_workspace(n))
    nat.call("xgs_vq_seed_farthest", nat.ptr(xt), dt, n, d, ldx, K, nat.ptr(seeds), nat.ptr(ws), ws.numel(),
             nat.stream_ptr())
    out = xt.index_select(0, seeds).to(t.float64)
    return to_host(out) if host else out


def warm_start(buffer, codebook: Codebook, cfg: VqConfig) -> WarmStartResult:
    """vq.py:150-170 — confidence-filtered hard-assignment initialisation."""
    t = nat.require_cuda()
    xt, dt, n, d, ldx = _rows(buffer)
    _check_d(d, codebook)
    if n == 0:
        raise InvalidInputError("warm-start buffer must be nonempty")
    host = _host_mode(buffer, codebook)
    E, K = _E(codebook), codebook.K
    if all_pass_provable(cfg.gamma, K):
        codes = _assign_dev(xt, dt, n, d, ldx, E, K)
        mask = None
        used = n
    else:
        _, _, codes, mask = _exact_dev(xt, dt, n, d, ldx, E, K, nat.EX_CODE | nat.EX_MASK, tau=cfg.tau_warm,
                                       gamma=cfg.gamma)
        used = int(mask.sum().item())
    if used == 0:
        return WarmStartResult(codebook=codebook, used=0, degenerate=True)
    counts, sums = _accumulate_dev(xt, dt, n, d, ldx, codes, mask, K)
    zero_cb = Codebook._make(E, t.zeros(K, dtype=t.float64, device="cuda"),
                             t.zeros((K, d), dtype=t.float64, device="cuda"), 0.0, codebook.epsilon,
                             codebook.reservoir)
    E2, N2, M2 = _ema_dev(zero_cb, counts, sums)  # lam = 0: N = c, M = s, E = M/(N+eps)
    if host:
        cb = Codebook(E=to_host(E2), N=to_host(N2), M=to_host(M2), lam=codebook.lam, epsilon=codebook.epsilon,
                      reservoir=codebook.reservoir)
    else:
        cb = Codebook._make(E2, N2, M2, codebook.lam, codebook.epsilon, codebook.reservoir)
    return WarmStartResult(codebook=cb, used=used, degenerate=False)


_pinned = threading.local()


def _small_to_host(t):
    """Read a small device tensor back through a reused pinned buffer (a
    pageable destination stages the copy through a driver buffer)."""
    torch = nat.torch()
    cache = getattr(_pinned, "bufs", None)
    if cache is None:
        cache = _pinned.bufs = {}
    key = (t.device.index, t.dtype, t.numel())
    buf = cache.get(key)
    if buf is None:
        buf = cache[key] = torch.empty(t.numel(), dtype=t.dtype, pin_memory=True)
    buf.copy_(t.reshape(-1), non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return buf.numpy().copy().reshape(tuple(t.shape))


def _revive_dev(codebook: Codebook, E, N, M, delta_dead, rng, N_host=None):
    """vq.py:173-190 on device tensors (E, N, M are updated in place)."""
    t = nat.torch()
    if N_host is None:
        N_host = _small_to_host(N)
    dead = np.nonzero(N_host < delta_dead)[0]
    if dead.size == 0:
        return [], False
    res = codebook.reservoir
    if len(res) == 0:
        return [], True
    rows = np.array([res._draw(rng) for _ in dead], dtype=np.int64)
    # the (dead code, ring row) pairs go to the device in one async copy from a
    # reused pinned buffer (two pageable copies had cost ~50 us per revival)
    nd = int(dead.size)
    hbuf, dbuf, ev = _revive_bufs(t, codebook.K)
    ev.synchronize()                      # the previous revival's copy has read the host buffer
    hbuf[:nd] = t.from_numpy(dead.astype(np.int64))
    hbuf[codebook.K:codebook.K + nd] = t.from_numpy(rows)
    dbuf.copy_(hbuf, non_blocking=True)
    ev.record()
    nat.call("xgs_vq_revive", codebook.K, codebook.D, float(codebook.epsilon), nat.ptr(res._ring), res.capacity,
             nat.ptr(dbuf), nat.ptr(dbuf[codebook.K:]), nd, nat.ptr(N), nat.ptr(M), nat.ptr(E), nat.stream_ptr())
    return [int(k) for k in dead], False


_REVIVE_BUFS = {}


def _revive_bufs(t, K):
    """Per (device, K): pinned host int64[2K], device int64[2K] and the event of
    the last copy out of the host buffer."""
    key = (t.cuda.current_device(), K)
    b = _REVIVE_BUFS.get(key)
    if b is None:
        b = (t.empty(2 * K, dtype=t.int64, pin_memory=True), t.empty(2 * K, dtype=t.int64, device="cuda"),
             t.cuda.Event())
        b[2].record()
        _REVIVE_BUFS[key] = b
    return b


def revive_dead_codes(codebook: Codebook, cfg: VqConfig, rng: np.random.Generator) -> ReviveResult:
    """vq.py:173-190 — reseed codes with N_k < delta from the reservoir."""
    host = _host_mode(codebook)
    N_host = to_host(codebook.N) if codebook.on_device else codebook.N
    if not np.any(N_host < cfg.delta_dead):
        return ReviveResult(codebook=codebook, revived=[], skipped=False)
    if len(codebook.reservoir) == 0:
        return ReviveResult(codebook=codebook, revived=[], skipped=True)
    E = device_f64(codebook.E, True).clone()
    N = device_f64(codebook.N).reshape(-1).clone()
    M = device_f64(codebook.M, True).clone()
    revived, skipped = _revive_dev(codebook, E, N, M, cfg.delta_dead, rng, N_host=N_host)
    if host:
        cb = Codebook(E=to_host(E), N=to_host(N), M=to_host(M), lam=codebook.lam, epsilon=codebook.epsilon,
                      reservoir=codebook.reservoir)
    else:
        cb = Codebook._make(E, N, M, codebook.lam, codebook.epsilon, codebook.reservoir)
    return ReviveResult(codebook=cb, revived=revived, skipped=skipped)


def local_stats(codebook: Codebook, xt, dt, n, d, ldx, cfg: VqConfig):
    """Per-shard half of online_step: mask + codes + (counts, sums) on device."""
    E, K = _E(codebook), codebook.K
    if all_pass_provable(cfg.gamma, K):
        _, counts, sums = _assign_accumulate_dev(xt, dt, n, d, ldx, E, K)
        return counts, sums
    else:
        _, _, codes, mask = _exact_dev(xt, dt, n, d, ldx, E, K, nat.EX_CODE | nat.EX_MASK, tau=cfg.tau_warm,
                                       gamma=cfg.gamma)
    return _accumulate_dev(xt, dt, n, d, ldx, codes, mask, K)


def online_step(codebook: Codebook, batch, cfg: VqConfig, rng: np.random.Generator):
    """vq.py:193-212 — one streaming update: reservoir insert, confidence
    filter, accumulate, EMA, revival.  Returns (Codebook, ReviveResult)."""
    xt, dt, n, d, ldx = _rows(batch)
    _check_d(d, codebook)
    if n == 0:
        raise InvalidInputError("batch must be nonempty")
    host = _host_mode(batch, codebook)
    codebook.reservoir._extend_rows(xt, dt, n, ldx)          # vq.py:203 (before the mask)
    counts, sums = local_stats(codebook, xt, dt, n, d, ldx, cfg)
    E, N, M = _ema_dev(codebook, counts, sums)
    revived, skipped = _revive_dev(codebook, E, N, M, cfg.delta_dead, rng)
    if host:
        cb = Codebook(E=to_host(E), N=to_host(N), M=to_host(M), lam=codebook.lam, epsilon=codebook.epsilon,
                      reservoir=codebook.reservoir)
    else:
        cb = Codebook._make(E, N, M, codebook.lam, codebook.epsilon, codebook.reservoir)
    return cb, ReviveResult(codebook=cb, revived=revived, skipped=skipped)


class VqAuditLog:
    """CSV audit trail for dead-code monitoring (vq.py:215-230)."""

    def __init__(self):
        self.rows = []

    def record(self, step: int, revived: Sequence[int], codebook: Codebook) -> None:
        N = to_host(codebook.N) if codebook.on_device else codebook.N
        self.rows.append((step, ";".join(str(i) for i in revived), float(N.min()) if codebook.K else 0.0,
                          float(N.max()) if codebook.K else 0.0))

    def write(self, path) -> None:
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["step", "revived_indices", "min_N", "max_N"])
            w.writerows(self.rows)
