"""TEST INFRASTRUCTURE ONLY — NumPy restatement of the reference's online EMA VQ.

Each function follows the reference function of the same name in
``/root/reference/pkg/src/semsplat/vq.py`` (cited per function) with the same
NumPy operations, so its results are bit-identical to the reference on the same
NumPy build (pinned by ``tests/golden`` vectors generated from the reference).
Row-chunking of the distance broadcast is bit-identical to the unchunked call
(each (row, code) value is an independent pairwise sum over D).

State is carried in :class:`OracleCodebook` (reference ``core.Codebook``,
core.py:206-243) and :class:`OracleReservoir` (reference
``core.FeatureReservoir``, core.py:178-203).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_CHUNK_BYTES = 256 << 20


class OracleReservoir:
    """Bounded FIFO of the most recent rows (core.py:178-203)."""

    def __init__(self, capacity: int, dim: int):
        self.capacity = int(capacity)
        self.dim = int(dim)
        self.buf = np.empty((0, dim), dtype=np.float64)

    def __len__(self):
        return self.buf.shape[0]

    def extend(self, x):  # core.py:191-195
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        self.buf = np.concatenate([self.buf, x])[-self.capacity:]

    def sample(self, rng):  # core.py:197-200
        return self.buf[int(rng.integers(0, len(self)))].copy()


@dataclass
class OracleCodebook:
    E: np.ndarray
    N: np.ndarray
    M: np.ndarray
    lam: float
    epsilon: float
    reservoir: OracleReservoir = field(default=None)

    def __post_init__(self):
        self.E = np.atleast_2d(np.asarray(self.E, dtype=np.float64))
        self.N = np.asarray(self.N, dtype=np.float64).reshape(-1)
        self.M = np.atleast_2d(np.asarray(self.M, dtype=np.float64))
        if self.reservoir is None:
            self.reservoir = OracleReservoir(4096, self.E.shape[1])

    @property
    def K(self):
        return self.E.shape[0]

    @property
    def D(self):
        return self.E.shape[1]

    def copy(self):
        return OracleCodebook(self.E.copy(), self.N.copy(), self.M.copy(), self.lam,
                              self.epsilon, self.reservoir)


def squared_distances(x, E):
    """vq.py:69-73 — (N,D)x(K,D) -> (N,K) by broadcast, pairwise sum over D."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    E = np.asarray(E, dtype=np.float64)
    n, K, D = x.shape[0], E.shape[0], E.shape[1]
    rows = max(1, _CHUNK_BYTES // max(1, K * D * 8))
    out = np.empty((n, K))
    for s in range(0, n, rows):
        diff = x[s:s + rows, None, :] - E[None, :, :]
        out[s:s + rows] = np.sum(diff * diff, axis=2)
    return out


def assign_batch(x, E):
    """vq.py:84-87 — np.argmin over the fp64 distances (first minimum)."""
    return np.argmin(squared_distances(x, E), axis=1)


def accumulate(batch, E):
    """vq.py:90-100 — counts = bincount(a), sums = np.add.at(zeros, a, batch)."""
    batch = np.atleast_2d(np.asarray(batch, dtype=np.float64))
    a = assign_batch(batch, E)
    K, D = E.shape
    counts = np.bincount(a, minlength=K).astype(np.float64)
    sums = np.zeros((K, D))
    np.add.at(sums, a, batch)
    return counts, sums


def ema_step(cb: OracleCodebook, counts, sums) -> OracleCodebook:
    """vq.py:103-109 — lam from the codebook, plain mul/add/div (no FMA)."""
    lam = cb.lam
    N = lam * cb.N + (1 - lam) * counts
    M = lam * cb.M + (1 - lam) * sums
    E = M / (N + cb.epsilon)[:, None]
    return OracleCodebook(E, N, M, cb.lam, cb.epsilon, cb.reservoir)


def confidence_scores(batch, E, tau):
    """vq.py:112-118 — softmax over -sqrt(d)/tau with the row-max shift."""
    d = np.sqrt(squared_distances(batch, E))
    logits = -d / tau
    logits -= logits.max(axis=1, keepdims=True)
    e = np.exp(logits)
    return e / e.sum(axis=1, keepdims=True)


def confidence_mask(batch, E, tau, gamma):
    """vq.py:121-124 — max softmax probability >= gamma."""
    return confidence_scores(batch, E, tau).max(axis=1) >= gamma


def seed_from_samples(buffer, K):
    """vq.py:127-147 — greedy farthest-point seeding."""
    buffer = np.atleast_2d(np.asarray(buffer, dtype=np.float64))
    seeds = [buffer[0]]
    min_d = np.sum((buffer - buffer[0]) ** 2, axis=1)
    while len(seeds) < K:
        j = int(np.argmax(min_d))
        if min_d[j] == 0.0:
            seeds.append(buffer[len(seeds) % buffer.shape[0]])
            continue
        seeds.append(buffer[j])
        min_d = np.minimum(min_d, np.sum((buffer - buffer[j]) ** 2, axis=1))
    return np.stack(seeds)


def warm_start(buffer, cb: OracleCodebook, tau, gamma):
    """vq.py:150-170 — confidence-filtered hard-assignment init (no EMA)."""
    buffer = np.atleast_2d(np.asarray(buffer, dtype=np.float64))
    mask = confidence_mask(buffer, cb.E, tau, gamma)
    used = int(mask.sum())
    if used == 0:
        return cb, 0, True
    kept = buffer[mask]
    a = assign_batch(kept, cb.E)
    N = np.bincount(a, minlength=cb.K).astype(np.float64)
    M = np.zeros_like(cb.M)
    np.add.at(M, a, kept)
    E = M / (N + cb.epsilon)[:, None]
    return OracleCodebook(E, N, M, cb.lam, cb.epsilon, cb.reservoir), used, False


def revive_dead_codes(cb: OracleCodebook, delta_dead, rng):
    """vq.py:173-190 — ascending dead k, one reservoir draw each."""
    dead = np.nonzero(cb.N < delta_dead)[0]
    if dead.size == 0:
        return cb, [], False
    if len(cb.reservoir) == 0:
        return cb, [], True
    N, M, E = cb.N.copy(), cb.M.copy(), cb.E.copy()
    for k in dead:
        x = cb.reservoir.sample(rng)
        M[k] = x
        N[k] = 1.0 + cb.epsilon
        E[k] = M[k] / (N[k] + cb.epsilon)
    return (OracleCodebook(E, N, M, cb.lam, cb.epsilon, cb.reservoir),
            [int(k) for k in dead], False)


def online_step(cb: OracleCodebook, batch, tau, gamma, delta_dead, rng, assume_all_pass=False):
    """vq.py:193-212 — reservoir extend, confidence filter, accumulate, EMA, revive.

    ``assume_all_pass`` skips the softmax when gamma <= fl(1/K), where the mask
    is provably all-true (max softmax >= 1/K); the result is identical.
    """
    batch = np.atleast_2d(np.asarray(batch, dtype=np.float64))
    cb.reservoir.extend(batch)
    if assume_all_pass:
        mask = np.ones(batch.shape[0], dtype=bool)
    else:
        mask = confidence_mask(batch, cb.E, tau, gamma)
    if mask.any():
        counts, sums = accumulate(batch[mask], cb.E)
    else:
        counts, sums = np.zeros(cb.K), np.zeros_like(cb.M)
    cb = ema_step(cb, counts, sums)
    return revive_dead_codes(cb, delta_dead, rng)
