"""CPU checks of the C-ABI boundary: libxgs.so loads without a GPU and exports
every entry point include/xgs.h declares; the ctypes table matches."""

import ctypes
import os
import re

from conftest import ROOT


def declared():
    src = open(os.path.join(ROOT, "include", "xgs.h")).read()
    return sorted(set(re.findall(r"XGS_API\s+[\w\s\*]+?\b(xgs_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    assert "xgs_vq_assign" in names and "xgs_vq_accumulate" in names and len(names) >= 10


def test_library_exports_every_declared_symbol():
    from paper_2603_09632_b200 import _native
    L = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing
    assert L.xgs_abi_version() == 2


def test_ctypes_table_matches_header():
    from paper_2603_09632_b200 import _native
    assert sorted(_native.SIGNATURES) == declared()
    _native.lib()  # binds every signature


def test_workspace_queries_without_gpu():
    from paper_2603_09632_b200 import _native
    L = _native.lib()
    assert L.xgs_vq_assign_workspace(1 << 20, 1024, 512, 0, 512) > (1 << 20) * 512 * 2
    assert L.xgs_vq_accumulate_workspace(1000, 16) > 4000


def test_screening_workspace_is_bounded_by_the_row_chunk():
    """The per-row screening buffers cover one row chunk (two slots), not the
    batch: at C5 on one GPU (67,108,864 bf16 rows x 1152, K=4096) the step
    workspace stays ~10 GB beside the 154.6 GB batch (it used to be another
    full fp16 copy of the batch plus N-sized queues)."""
    from paper_2603_09632_b200 import _native
    L = _native.lib()
    n, k, d = 67_108_864, 4096, 1152
    step = L.xgs_vq_step_workspace(n, k, d, 2, d)
    assert step < 12e9, step
    small = L.xgs_vq_step_workspace(1 << 22, k, d, 2, d)
    big = L.xgs_vq_step_workspace(1 << 24, k, d, 2, d)
    # beyond one chunk the screening part is flat; only the 4-byte-per-row accumulate part grows
    assert big - small < (1 << 24) * 16


def test_error_codes_map_to_reference_exceptions():
    """Argument validation happens before any CUDA call, so the status codes
    and the InvalidInputError / InvalidStateError mapping are checkable here."""
    import ctypes

    import pytest

    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.errors import InvalidInputError, InvalidStateError
    L = nat.lib()
    dummy = ctypes.c_void_p(16)
    # K == 0 -> invalid state (vq.py:85-86)
    rc = L.xgs_vq_assign(dummy, 0, 4, 3, 3, dummy, 0, dummy, dummy, 1 << 30, None, None)
    assert rc == 2 and b"empty codebook" in L.xgs_last_error()
    with pytest.raises(InvalidStateError):
        nat.check(rc)
    # bad dtype / shape / ldx < d -> invalid input
    assert L.xgs_vq_assign(dummy, 7, 4, 3, 3, dummy, 5, dummy, dummy, 1 << 30, None, None) == 1
    assert L.xgs_vq_assign(dummy, 0, 4, 3, 2, dummy, 5, dummy, dummy, 1 << 30, None, None) == 1
    with pytest.raises(InvalidInputError):
        nat.check(1)
    # workspace too small
    assert L.xgs_vq_assign(dummy, 0, 4, 3, 3, dummy, 5, dummy, dummy, 16, None, None) == 1
    # EMA decay outside [0, 1) (core.py:223-224)
    assert L.xgs_vq_ema(1.0, 1e-5, 2, 2, dummy, dummy, dummy, dummy, dummy, dummy, dummy, None) == 1
    # ring write larger than the capacity
    assert L.xgs_vq_ring_write(dummy, 0, 3, 0, 10, 3, dummy, 4, 0, None) == 1
    # grid: non-positive voxel / bad mode
    fr = nat.GridFrames(1, 4, 4, 16, None, 16, 16, 1.0, 1.0, 0.0, 0.0, 0.0, 1, 0, 1e-3, None, 0, 0, 0)
    res = nat.GridResult(16, 16, 16, 16, 16, 16, 16, None, 16, 0, 0, 0, 0, 0)
    assert L.xgs_grid_sample(ctypes.byref(fr), dummy, ctypes.byref(res), dummy, 1 << 30, None) == 1
    fr.voxel, fr.mode = 0.1, 3
    assert L.xgs_grid_sample(ctypes.byref(fr), dummy, ctypes.byref(res), dummy, 1 << 30, None) == 1


def test_python_api_validation_without_gpu():
    import numpy as np
    import pytest

    import paper_2603_09632_b200 as xv
    with pytest.raises(xv.InvalidInputError):
        xv.VqConfig(lam=1.0)
    with pytest.raises(xv.InvalidInputError):
        xv.VqConfig(gamma=0.0)
    with pytest.raises(xv.InvalidInputError):
        xv.VqConfig(K=0)
    with pytest.raises(xv.InvalidInputError):
        xv.Codebook(E=np.zeros((3, 2)), N=np.zeros(2), M=np.zeros((3, 2)), lam=0.5, epsilon=1e-5)
    with pytest.raises(xv.InvalidInputError):
        xv.Codebook(E=np.zeros((2, 2)), N=-np.ones(2), M=np.zeros((2, 2)), lam=0.5, epsilon=1e-5)
    with pytest.raises(xv.InvalidInputError):
        xv.FeatureReservoir(0, 3)
    with pytest.raises(xv.InvalidInputError):
        xv.CameraPose(np.diag([1.0, 1.0, -1.0]), np.zeros(3))
