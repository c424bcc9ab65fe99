"""ctypes binding of libxgs.so (the C ABI in include/xgs.h).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises :class:`NativeError`.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import InvalidInputError, InvalidStateError, NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libxgs.so")

F32, F64, BF16 = 0, 1, 2
GRID_ASYNC = 1
EX_DIST, EX_CODE, EX_MASK, EX_PROB = 1, 2, 4, 8

_lib = None
_lock = threading.Lock()

_vp, _i64, _i32, _f64, _sz = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                              ctypes.c_size_t)

# name -> (restype, argtypes); mirrors include/xgs.h
SIGNATURES = {
    "xgs_abi_version": (_i32, []),
    "xgs_last_error": (ctypes.c_char_p, []),
    "xgs_device_sm_count": (_i32, []),
    "xgs_launch_count": (ctypes.c_longlong, []),
    "xgs_profile_enable": (_i32, [_i32]),
    "xgs_profile_only": (_i32, [ctypes.c_char_p]),
    "xgs_profile_read": (_i32, [ctypes.c_char_p, _vp, _vp]),
    "xgs_profile_dump": (_i32, [ctypes.c_char_p]),
    "xgs_vq_assign_workspace": (_sz, [_i64, _i64, _i64, _i32, _i64]),
    "xgs_vq_assign": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp, _vp]),
    "xgs_vq_assign_dev": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _sz, _vp, _vp]),
    "xgs_vq_exact": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _i32, _f64, _f64, _vp, _vp, _vp, _vp,
                            _vp]),
    "xgs_vq_step_workspace": (_sz, [_i64, _i64, _i64, _i32, _i64]),
    "xgs_vq_assign_accumulate": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz, _vp,
                                        _vp]),
    "xgs_vq_assign_accumulate_h2d": (_i32, [_vp, _vp, _i32, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp, _sz,
                                            _vp, _vp]),
    "xgs_vq_accumulate_workspace": (_sz, [_i64, _i64]),
    "xgs_vq_seed_workspace": (_sz, [_i64]),
    "xgs_vq_seed_farthest": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _vp, _sz, _vp]),
    "xgs_vq_accumulate": (_i32, [_vp, _i32, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _sz, _vp]),
    "xgs_vq_ema": (_i32, [_f64, _f64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "xgs_vq_revive": (_i32, [_i64, _i64, _f64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "xgs_vq_ring_write": (_i32, [_vp, _i32, _i64, _i64, _i64, _i64, _vp, _i64, _i64, _vp]),
    "xgs_vq_ring_write_dev": (_i32, [_vp, _i32, _i64, _vp, _i64, _i64, _vp, _i64, _vp, _vp]),
    "xgs_gather_rows_f64": (_i32, [_vp, _i64, _vp, _i64, _vp, _vp]),
    "xgs_backproject": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "xgs_hashset_create": (_i32, [_i64, _vp]),
    "xgs_hashset_destroy": (_i32, [_vp]),
    "xgs_hashset_insert": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "xgs_hashset_contains": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "xgs_hashset_size": (_i32, [_vp, _vp, _vp]),
    "xgs_hashset_copy": (_i32, [_vp, _vp, _vp]),
    "xgs_grid_workspace": (_sz, [_i64]),
    "xgs_radix_sort_pairs_u64": (_i32, [_vp, _vp, _i64, _i32, _vp, _sz, _vp]),
    "xgs_grid_sample": (_i32, [_vp, _vp, _vp, _vp, _sz, _vp]),
    "xgs_grid_sample_h2d": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "xgs_prefix_mask": (_i32, [_vp, _i64, _vp, _vp]),
    "xgs_pose_depths": (_i32, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "xgs_gemm_f64_workspace": (_sz, [_i64, _i64, _i64, _i64, _i32]),
    "xgs_gemm_f64": (_i32, [_vp, _i64, _i64, _i64, _i64, _i32, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _f64,
                            _f64, _vp, _vp, _sz, _vp]),
    "xgs_sup_gather": (_i32, [_vp, _i32, _i64, _i64, _vp, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _i64,
                              _i64, _vp, _vp, _vp, _vp]),
    "xgs_sup_loss": (_i32, [_vp, _vp, _vp, _i64, _i64, _f64, _vp, _vp, _vp]),
    "xgs_softmax_rows": (_i32, [_vp, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "xgs_raster_build": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "xgs_raster_fetch": (_i32, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "xgs_raster_accumulate": (_i32, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "xgs_raster_argmax": (_i32, [_vp, _vp, _vp]),
    "xgs_raster_vjp": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "xgs_raster_free": (_i32, [_vp]),
    "xgs_contrast_scores": (_i32, [_vp, _i64, _i64, _vp, _i64, _f64, _f64, _vp, _vp]),
    "xgs_desc_order_keys": (_i32, [_vp, _i64, _vp, _vp, _vp]),
    "xgs_desc_top_m_workspace": (_sz, [_i64]),
    "xgs_desc_top_m": (_i32, [_vp, _i64, _i64, _vp, _vp, _sz, _vp]),
}


class GridFrames(ctypes.Structure):
    """Mirror of xgs_grid_frames (include/xgs.h)."""
    _fields_ = [("frames", _i64), ("height", _i64), ("width", _i64), ("depth", _vp), ("color", _vp),
                ("rot", _vp), ("trans", _vp), ("fx", _f64), ("fy", _f64), ("cx", _f64), ("cy", _f64),
                ("voxel", _f64), ("stride", ctypes.c_int32), ("mode", ctypes.c_int32), ("min_scale", _f64),
                ("feat", _vp), ("feat_c", _i64), ("feat_h", _i64), ("feat_w", _i64), ("flags", ctypes.c_int32)]


class GridResult(ctypes.Structure):
    """Mirror of xgs_grid_result (include/xgs.h)."""
    _fields_ = [("capacity", _i64), ("key", _vp), ("pid", _vp), ("mu", _vp), ("color", _vp), ("scale", _vp),
                ("depth", _vp), ("feat", _vp), ("count", _vp), ("n_new", _i64), ("n_valid", _i64),
                ("n_voxels", _i64), ("n_sorted", _i64), ("sort_passes", _i64), ("feat_dtype", ctypes.c_int32),
                ("dev_status", _vp)]


class RasterIn(ctypes.Structure):
    """Mirror of xgs_raster_in (include/xgs.h)."""
    _fields_ = [("n", _i64), ("mu", _vp), ("quat", _vp), ("scale", _vp), ("opacity", _vp),
                ("R", _f64 * 9), ("t", _f64 * 3), ("fx", _f64), ("fy", _f64), ("cx", _f64), ("cy", _f64),
                ("near_z", _f64), ("far_z", _f64), ("n_rows", _i64), ("row0", _i64), ("row_step", _i64),
                ("n_cols", _i64), ("col0", _i64), ("col_step", _i64), ("term_threshold", _f64),
                ("cutoff_sigma", _f64), ("eig_floor", _f64), ("all_pairs", ctypes.c_int32)]


def lib():
    """Load libxgs.so (raises NativeError when it was not built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeError(f"libxgs.so not built ({LIB_PATH}); run "
                                      "`python -m paper_2603_09632_b200.build`")
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def launch_count():
    return int(lib().xgs_launch_count())


def profile_enable(on=True):
    check(lib().xgs_profile_enable(1 if on else 0))


def profile_only(tag=None):
    """Record only scopes named `tag` (None: all)."""
    check(lib().xgs_profile_only(tag.encode() if tag else None))


def profile_read(tag):
    ms, cnt = ctypes.c_double(0), ctypes.c_longlong(0)
    check(lib().xgs_profile_read(tag.encode(), ctypes.byref(ms), ctypes.byref(cnt)))
    return ms.value, cnt.value


def check(rc):
    if rc == 0:
        return
    msg = lib().xgs_last_error().decode(errors="replace")
    if rc == 1:
        raise InvalidInputError(msg)
    if rc == 2:
        raise InvalidStateError(msg)
    raise NativeError(f"libxgs error {rc}: {msg}")


def call(name, *args):
    check(getattr(lib(), name)(*args))


# ---------------------------------------------------------------- torch glue

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise NativeError("no CUDA device visible: the B200 path has no CPU fallback")
    lib()
    return t


def stream_ptr():
    """The current CUDA stream of the current device (raw handle; the torch.cuda
    Stream object costs ~6 us per query, this ~1 us -- it is on every call)."""
    C = torch()._C
    return ctypes.c_void_p(C._cuda_getCurrentRawStream(C._cuda_getDevice()))


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


_ws = {}


def workspace(slot, nbytes, device=None):
    """Grow-only per-(device, slot) scratch buffer (uint8 CUDA tensor)."""
    t = torch()
    dev = t.device("cuda", t.cuda.current_device()) if device is None else device
    key = (dev.index, slot)
    buf = _ws.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = t.empty(max(int(nbytes), 256), dtype=t.uint8, device=dev)
        _ws[key] = buf
    return buf


def dtype_code(tensor):
    t = torch()
    if tensor.dtype == t.float32:
        return F32
    if tensor.dtype == t.float64:
        return F64
    if tensor.dtype == t.bfloat16:
        return BF16
    raise InvalidInputError(f"unsupported dtype {tensor.dtype}")
