"""Host-side logic of the reference shim (no GPU): install / uninstall rebinding,
the host FIFO update that mirrors FeatureReservoir.extend (core.py:191-195),
error translation to the reference's classes, and type detection.  Skipped
when the reference is not installed under baseline/_ref."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "semsplat")),
                                reason="reference not installed under baseline/_ref")


@pytest.fixture()
def ref():
    sys.path.insert(0, REF)
    import semsplat.core as rc
    import semsplat.errors as re_
    import semsplat.slam as rs
    import semsplat.vq as rv
    yield rc, rv, re_, rs
    sys.path.remove(REF)


def test_install_rebinds_and_uninstall_restores(ref):
    rc, rv, re_, rs = ref
    from paper_2603_09632_b200 import reference_shim as sh
    orig = {n: getattr(rv, n) for n in sh.VQ_FUNCS}
    names = sh.install()
    try:
        assert len(names) == len(sh.VQ_FUNCS) + len(sh.SLAM_FUNCS)
        for n in sh.VQ_FUNCS:
            assert getattr(rv, n) is not orig[n] and getattr(rv, n).__b200__
            assert getattr(rv, n).__wrapped_reference__ is orig[n]
        assert sh.install() == names          # idempotent
    finally:
        sh.uninstall()
    for n in sh.VQ_FUNCS:
        assert getattr(rv, n) is orig[n]


@pytest.mark.parametrize("cap,batches", [(5, [3, 4, 1]), (4, [10]), (6, [2, 2, 2, 2])])
def test_host_fifo_matches_reference_extend(ref, cap, batches):
    rc, _, _, _ = ref
    from paper_2603_09632_b200 import reference_shim as sh
    rng = np.random.default_rng(cap)
    a, b = rc.FeatureReservoir(cap, 3), rc.FeatureReservoir(cap, 3)
    sh._mirrors[b] = [None, b._buf]        # as if mirrored (no device needed for the host half)
    for n in batches:
        x = rng.normal(size=(n, 3)).astype(np.float32)
        a.extend(x)                          # the reference
        sh._push_host(b, x)                  # the shim's host update
        assert np.array_equal(a.as_array(), b.as_array())
        assert sh._mirrors[b][1] is b._buf   # version stamp follows the rebinding


def test_error_translation_and_type_detection(ref):
    rc, _, re_, _ = ref
    from paper_2603_09632_b200 import errors as xe
    from paper_2603_09632_b200 import reference_shim as sh

    def boom():
        raise xe.InvalidInputError("dimension mismatch")

    with pytest.raises(re_.InvalidInputError, match="dimension mismatch"):
        sh._translate(boom)()

    def boom2():
        raise xe.InvalidStateError("empty")

    with pytest.raises(re_.InvalidStateError):
        sh._translate(boom2)()
    cb = rc.Codebook(E=np.eye(2), N=np.zeros(2), M=np.zeros((2, 2)), lam=0.5, epsilon=1e-5)
    assert sh._is_ref_codebook(cb)
    from paper_2603_09632_b200.core import Codebook
    assert not sh._is_ref_codebook(Codebook(E=np.eye(2), N=np.zeros(2), M=np.zeros((2, 2)), lam=0.5, epsilon=1e-5))
