"""Install the B200 path under an existing ``semsplat`` installation.

The reference's boundary for the hot path is its Python API:
``semsplat.vq`` (vq.py:62-212) and ``semsplat.slam.backproject`` /
``densify_and_prune`` (slam.py:594-651).  :func:`install` rebinds those module
attributes to adapters over this package, so every caller that looks the
functions up through the module -- including ``from semsplat.vq import
online_step`` executed after ``install()`` -- runs on the B200 with the
reference's own types:

* ``semsplat.core.Codebook`` in -> ``semsplat.core.Codebook`` out
  (core.py:206-243), built with the reference class, sharing the caller's
  ``FeatureReservoir`` object;
* ``semsplat.core.FeatureReservoir`` (core.py:178-203) keeps its own host FIFO
  (``_buf``) exactly as the reference maintains it; a device mirror ring
  (``core.FeatureReservoir``) serves the revival gathers.  The mirror is
  re-uploaded whenever the host FIFO was changed behind the shim's back
  (``reservoir.extend`` called directly -- the reference rebinds ``_buf`` on
  every extend, so identity of the array is the version stamp);
* result records are the reference's ``VqBatchStats`` / ``WarmStartResult`` /
  ``ReviveResult`` (vq.py:42-59) and ``GaussianField`` (core.py:107-175);
* errors surface as the reference's ``semsplat.errors`` classes
  (errors.py:8-21), so ``except semsplat.errors.InvalidInputError`` keeps
  working.

``uninstall()`` restores the original attributes.  The reference package is
never imported by this module at import time; it is located at install time
(``import semsplat``) -- in this repository that is the pip install under
``baseline/_ref`` (tools/install_reference.sh).
"""

from __future__ import annotations

import functools
import importlib
import weakref

import numpy as np

from . import core as xcore
from . import errors as xerr
from . import slam as xslam
from . import vq as xvq

VQ_FUNCS = ("squared_distances", "assign", "assign_batch", "accumulate", "ema_step", "confidence_scores",
            "confidence_mask", "seed_from_samples", "warm_start", "revive_dead_codes", "online_step")
SLAM_FUNCS = ("backproject", "densify_and_prune")

_saved = {}
_mirrors = weakref.WeakKeyDictionary()   # reference FeatureReservoir -> [device mirror, synced _buf]


def _ref():
    rc = importlib.import_module("semsplat.core")
    rv = importlib.import_module("semsplat.vq")
    re_ = importlib.import_module("semsplat.errors")
    rs = importlib.import_module("semsplat.slam")
    return rc, rv, re_, rs


# ------------------------------------------------------------ type adapters

def _mirror(res):
    """Device ring mirroring a reference FeatureReservoir (re-synced when the
    host FIFO array changed identity)."""
    if res is None or isinstance(res, xcore.FeatureReservoir):
        return res
    ent = _mirrors.get(res)
    if ent is None:
        ent = [xcore.FeatureReservoir(res.capacity, res.dim), None]
        _mirrors[res] = ent
    mir, synced = ent
    if synced is not res._buf:
        buf = np.ascontiguousarray(res._buf, dtype=np.float64)
        mir._head, mir._len = 0, 0
        if buf.shape[0]:
            mir.extend(buf)
        ent[1] = res._buf
    return mir


def _push_host(res, batch):
    """The reference FIFO update of vq.py:203 (core.py:191-195) on the host
    copy, touching only the rows that can survive (the last ``capacity``)."""
    if res is None or isinstance(res, xcore.FeatureReservoir):
        return
    b = batch.detach().cpu().numpy() if xcore.is_tensor(batch) else batch
    tail = np.atleast_2d(np.asarray(b, dtype=np.float64))[-res.capacity:]
    res._buf = np.concatenate([res._buf, tail])[-res.capacity:]
    _mirrors[res][1] = res._buf


def _is_ref_codebook(cb):
    return cb is not None and not isinstance(cb, xcore.Codebook) and hasattr(cb, "E") and hasattr(cb, "reservoir")


def _to_x(cb):
    """Reference Codebook -> this package's Codebook over the same arrays."""
    if not _is_ref_codebook(cb):
        return cb
    return xcore.Codebook._make(np.asarray(cb.E, dtype=np.float64), np.asarray(cb.N, dtype=np.float64).reshape(-1),
                                np.asarray(cb.M, dtype=np.float64), float(cb.lam), float(cb.epsilon),
                                _mirror(cb.reservoir))


def _to_ref(xcb, like):
    """This package's Codebook -> reference Codebook carrying ``like``'s reservoir."""
    rc = _ref()[0]
    c = xcb.to_numpy()
    return rc.Codebook(E=c.E, N=c.N, M=c.M, lam=c.lam, epsilon=c.epsilon, reservoir=like.reservoir)


def _translate(fn):
    """Re-raise this package's errors as the reference's classes (same name)."""
    @functools.wraps(fn)
    def wrapper(*a, **k):
        try:
            return fn(*a, **k)
        except xerr.SemsplatError as e:
            re_ = _ref()[2]
            cls = getattr(re_, type(e).__name__, None)
            if cls is None or not isinstance(cls, type) or not issubclass(cls, Exception):
                raise
            raise cls(str(e)) from e
    return wrapper


# ------------------------------------------------------------ VQ adapters (vq.py:62-212)

def _squared_distances(x, codebook):
    return xvq.squared_distances(x, _to_x(codebook))


def _assign(x, codebook):
    return xvq.assign(x, _to_x(codebook))


def _assign_batch(x, codebook):
    return xvq.assign_batch(x, _to_x(codebook))


def _accumulate(batch, codebook):
    rv = _ref()[1]
    st = xvq.accumulate(batch, _to_x(codebook))
    return rv.VqBatchStats(counts=st.counts, sums=st.sums) if _is_ref_codebook(codebook) else st


def _ema_step(codebook, stats):
    out = xvq.ema_step(_to_x(codebook), stats)
    return _to_ref(out, codebook) if _is_ref_codebook(codebook) else out


def _confidence_scores(batch, codebook, tau):
    return xvq.confidence_scores(batch, _to_x(codebook), tau)


def _confidence_mask(batch, codebook, cfg):
    return xvq.confidence_mask(batch, _to_x(codebook), cfg)


def _seed_from_samples(buffer, K):
    return xvq.seed_from_samples(buffer, K)


def _warm_start(buffer, codebook, cfg):
    res = xvq.warm_start(buffer, _to_x(codebook), cfg)
    if not _is_ref_codebook(codebook):
        return res
    rv = _ref()[1]
    cb = codebook if res.degenerate else _to_ref(res.codebook, codebook)
    return rv.WarmStartResult(codebook=cb, used=res.used, degenerate=res.degenerate)


def _revive_dead_codes(codebook, cfg, rng):
    res = xvq.revive_dead_codes(_to_x(codebook), cfg, rng)
    if not _is_ref_codebook(codebook):
        return res
    rv = _ref()[1]
    cb = _to_ref(res.codebook, codebook) if res.revived else codebook
    return rv.ReviveResult(codebook=cb, revived=res.revived, skipped=res.skipped)


def _online_step(codebook, batch, cfg, rng):
    if not _is_ref_codebook(codebook):
        return xvq.online_step(codebook, batch, cfg, rng)
    rv = _ref()[1]
    xcb = _to_x(codebook)
    out, res = xvq.online_step(xcb, batch, cfg, rng)   # extends the device mirror (vq.py:203)
    _push_host(codebook.reservoir, batch)               # ... and the reference's host FIFO alike
    cb = _to_ref(out, codebook)
    return cb, rv.ReviveResult(codebook=cb, revived=res.revived, skipped=res.skipped)


# ------------------------------------------------------------ SLAM adapters (slam.py:594-651)

def _backproject(pose, intr, u, v, depth):
    return xslam.backproject(pose, intr, u, v, depth)


def _densify_and_prune(field_, window, cfg, K=None):
    rc = _ref()[0]
    out = xslam.densify_and_prune(field_, window, cfg, K)
    if out is field_ or isinstance(out, rc.GaussianField):
        return out
    return rc.GaussianField(mu=out.mu, quat=out.quat, scale=out.scale, opacity=out.opacity, color=out.color,
                            logits=out.logits, generation=out.generation)


_ADAPTERS = {
    "squared_distances": _squared_distances, "assign": _assign, "assign_batch": _assign_batch,
    "accumulate": _accumulate, "ema_step": _ema_step, "confidence_scores": _confidence_scores,
    "confidence_mask": _confidence_mask, "seed_from_samples": _seed_from_samples, "warm_start": _warm_start,
    "revive_dead_codes": _revive_dead_codes, "online_step": _online_step,
    "backproject": _backproject, "densify_and_prune": _densify_and_prune,
}


def install(slam: bool = True):
    """Rebind ``semsplat.vq`` (and ``semsplat.slam``'s back-projection /
    insertion) to the B200 path.  Idempotent; returns the names installed."""
    rc, rv, re_, rs = _ref()
    done = []
    targets = [(rv, VQ_FUNCS)] + ([(rs, SLAM_FUNCS)] if slam else [])
    for mod, names in targets:
        for name in names:
            key = (mod.__name__, name)
            if key not in _saved:
                _saved[key] = getattr(mod, name)
            fn = _translate(_ADAPTERS[name])
            fn.__b200__ = True
            fn.__wrapped_reference__ = _saved[key]
            setattr(mod, name, fn)
            done.append(f"{mod.__name__}.{name}")
    return done


def uninstall():
    for (modname, name), fn in list(_saved.items()):
        setattr(importlib.import_module(modname), name, fn)
    _saved.clear()
