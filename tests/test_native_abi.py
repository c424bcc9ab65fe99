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
    assert L.xgs_abi_version() == 1


def test_ctypes_table_matches_header():
    from paper_2603_09632_b200 import _native
    assert sorted(_native.SIGNATURES) == declared()
    _native.lib()  # binds every signature


def test_workspace_queries_without_gpu():
    from paper_2603_09632_b200 import _native
    L = _native.lib()
    assert L.xgs_vq_assign_workspace(1 << 20, 1024, 512, 0, 512) > (1 << 20) * 512 * 2
    assert L.xgs_vq_accumulate_workspace(1000, 16) > 4000
