"""TEST INFRASTRUCTURE ONLY — NumPy restatement of the codebook consumers
(reference pkg/src/semsplat/core.py:473-496 and thinker.py:110-206), pinned by
tests/golden/thinker.npz (generated from the reference)."""

from __future__ import annotations

import numpy as np

NORM_EPS = 1e-8


def mixture_weights(L):                                   # core.py:473-480
    L = np.asarray(L, dtype=np.float64)
    e = np.exp(L - np.max(L, axis=-1, keepdims=True))
    return e / np.sum(e, axis=-1, keepdims=True)


def softmax_vjp(L, up):                                   # core.py:483-487
    w = mixture_weights(L)
    return w * (up - np.sum(w * up, axis=-1, keepdims=True))


def decode_feature(L, E):                                 # core.py:490-496
    return mixture_weights(L) @ E


def semantic_entropy(L):                                  # thinker.py:185-191
    p = mixture_weights(np.atleast_2d(L))
    with np.errstate(divide="ignore", invalid="ignore"):
        plogp = np.where(p > 0, p * np.log(p), 0.0)
    return -np.sum(plogp, axis=-1)


def contrast_scores(F, pos, negs, tau):                   # thinker.py:110-119, :128-129
    Fu = F / (np.linalg.norm(F, axis=1, keepdims=True) + NORM_EPS)
    p = Fu @ pos
    s = np.ones(F.shape[0])
    for n in negs:
        s = np.minimum(s, 1.0 / (1.0 + np.exp(-tau * (p - Fu @ n))))
    return s


def mask_gaussians(scores, delta, fallback_frac=0.01):     # thinker.py:159-174
    m = scores > delta
    if m.any():
        return m, False
    k = max(1, int(np.ceil(fallback_frac * scores.size)))
    m = np.zeros(scores.size, dtype=bool)
    m[np.argsort(-scores, kind="stable")[:k]] = True
    return m, True


def sample_tokens(L, E, M):                                # thinker.py:194-206
    H = semantic_entropy(L)
    o = np.argsort(-H, kind="stable")[:min(M, L.shape[0])]
    return o, H[o], decode_feature(L[o], E)
