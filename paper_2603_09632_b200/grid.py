"""GPU voxel grid sampling of back-projected RGB-D frames (north-star GRID half).

The reference has no voxel sampler: its only code that turns back-projected
RGB-D pixels into new Gaussians is ``slam.backproject`` + the insertion half
of ``slam.densify_and_prune`` (slam.py:594-651).  This module keeps that
arithmetic and conventions (fp64 back-projection in the reference's operation
order, ``depth > 0`` validity, stride lattice, rgb/255 colours, iso size
``max(min_scale, 0.5*s*depth/fx)``, row-major emission) and replaces the
per-pixel Python loop + coverage render with the libxgs pipeline
(include/xgs.h ``xgs_grid_sample``): keys -> in-house LSD radix sort ->
first-pick / mean select -> hash-set occupancy test -> pixel-order emit.
Definitions: SURVEY.md §8(a) g8, oracle/grid.py.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _native as nat
from .core import CameraIntrinsics, CameraPose, is_tensor
from .errors import InvalidInputError, InvalidStateError

KEY_BIAS = 1 << 20
KEY_INVALID = (1 << 64) - 1


def pack_key(ix, iy, iz):
    """Voxel indices -> 63-bit keys (21-bit fields biased by 2^20)."""
    ix, iy, iz = (np.asarray(a, dtype=np.int64) + KEY_BIAS for a in (ix, iy, iz))
    return ((ix.astype(np.uint64) << np.uint64(42)) | (iy.astype(np.uint64) << np.uint64(21))
            | iz.astype(np.uint64))


class VoxelHashSet:
    """Occupied-voxel set of the map, resident in HBM (open addressing)."""

    def __init__(self, capacity: int = 1 << 20):
        nat.require_cuda()
        h = ctypes.c_void_p()
        nat.call("xgs_hashset_create", int(capacity), ctypes.byref(h))
        self._h = h

    def __len__(self):
        n = ctypes.c_int64()
        nat.call("xgs_hashset_size", self._h, ctypes.byref(n), nat.stream_ptr())
        return int(n.value)

    def _keys(self, keys):
        t = nat.torch()
        if not is_tensor(keys):
            keys = t.from_numpy(np.ascontiguousarray(np.asarray(keys, dtype=np.uint64)).view(np.int64))
        return keys.to(device="cuda", dtype=t.int64).contiguous()

    def insert(self, keys):
        """Insert-if-absent; returns a bool mask of keys that were new."""
        t = nat.torch()
        k = self._keys(keys)
        out = t.empty(k.numel(), dtype=t.uint8, device="cuda")
        nat.call("xgs_hashset_insert", self._h, nat.ptr(k), k.numel(), nat.ptr(out), nat.stream_ptr())
        return out.bool()

    def contains(self, keys):
        t = nat.torch()
        k = self._keys(keys)
        out = t.empty(k.numel(), dtype=t.uint8, device="cuda")
        nat.call("xgs_hashset_contains", self._h, nat.ptr(k), k.numel(), nat.ptr(out), nat.stream_ptr())
        return out.bool()

    def copy_from(self, other: "VoxelHashSet"):
        """Snapshot / restore: this set's keys become `other`'s (stream-ordered;
        both created with the same capacity and not grown since)."""
        nat.call("xgs_hashset_copy", self._h, other._h, nat.stream_ptr())
        return self

    def close(self):
        if getattr(self, "_h", None) is not None and nat._lib is not None:
            nat.lib().xgs_hashset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GridSampleResult:
    """New Gaussians of one batch, ascending (frame, pixel) id (CUDA tensors).

    The fields are views of the call's output buffer, created on first access
    (a batch that only needs counts, or goes straight to ``to_numpy``, builds
    no per-field tensor views on the host):

    key      (n,) int64 view of the uint64 voxel keys
    pid      (n,) int64: frame*H*W + u*W + v
    mu       (n, 3) fp64 world positions
    color    (n, 3) fp64 rgb/255
    scale    (n,) fp64 iso size
    depth    (n,) fp64 camera depth of the representative pixel
    count    (n,) fp64 points averaged (mean mode) or 1
    feature  (n, C) fp32 (first-pick) / fp64 (mean) or None
    """

    __slots__ = ("_flat", "_cap", "_n", "_feat", "n_valid", "n_voxels", "n_sorted", "sort_passes", "_cache")

    def __init__(self, flat, cap, n, feat, n_valid, n_voxels, n_sorted=0, sort_passes=0):
        self._flat, self._cap, self._n, self._feat = flat, cap, n, feat
        self.n_valid, self.n_voxels, self.n_sorted, self.sort_passes = n_valid, n_voxels, n_sorted, sort_passes
        self._cache = {}

    def __len__(self):
        return self._n

    def _col(self, name):
        v = self._cache.get(name)
        if v is None:
            t = nat.torch()
            f, c, n = self._flat, self._cap, self._n
            v = {"key": lambda: f[:n].view(t.int64), "pid": lambda: f[c:c + n].view(t.int64),
                 "mu": lambda: f[2 * c:2 * c + 3 * n].view(n, 3), "color": lambda: f[5 * c:5 * c + 3 * n].view(n, 3),
                 "scale": lambda: f[8 * c:8 * c + n], "depth": lambda: f[9 * c:9 * c + n],
                 "count": lambda: f[10 * c:10 * c + n]}[name]()
            self._cache[name] = v
        return v

    key = property(lambda self: self._col("key"))
    pid = property(lambda self: self._col("pid"))
    mu = property(lambda self: self._col("mu"))
    color = property(lambda self: self._col("color"))
    scale = property(lambda self: self._col("scale"))
    depth = property(lambda self: self._col("depth"))
    count = property(lambda self: self._col("count"))

    @property
    def feature(self):
        return None if self._feat is None else self._feat[:self._n]

    def to_numpy(self):
        """All fields in ONE device->host copy: the per-voxel columns are packed
        into one device buffer (a few µs) and read back through a reused
        pinned landing buffer (8 pageable copies would each stage through a
        driver buffer and run at about half the PCIe rate)."""
        t = nat.torch()
        n, c, f = self._n, self._cap, self._flat
        cols = [f[:2 * n] if c == n else t.cat([f[:n], f[c:c + n]]) if n else f[:0]]
        cols += [f[2 * c:2 * c + 3 * n], f[5 * c:5 * c + 3 * n], f[8 * c:8 * c + n], f[9 * c:9 * c + n],
                 f[10 * c:10 * c + n]]
        feat = self.feature
        if feat is not None:
            cols.append(feat.reshape(-1) if feat.dtype == t.float64 else
                        feat.reshape(-1).view(t.int32).to(t.float64))    # fp32 bits carried losslessly
        packed = t.cat(cols) if n else t.empty(0, dtype=t.float64, device="cuda")
        host = _pinned_landing(packed.numel())
        host[:packed.numel()].copy_(packed, non_blocking=True)
        t.cuda.current_stream().synchronize()
        a = host[:packed.numel()].numpy().copy()
        o = [0]

        def take(m):
            r = a[o[0]:o[0] + m]
            o[0] += m
            return r
        out = dict(key=take(n).view(np.uint64), pid=take(n).view(np.int64), mu=take(3 * n).reshape(n, 3),
                   color=take(3 * n).reshape(n, 3), scale=take(n), depth=take(n), count=take(n), feature=None,
                   n_valid=self.n_valid, n_voxels=self.n_voxels, n_sorted=self.n_sorted,
                   sort_passes=self.sort_passes)
        if feat is not None:
            C = int(feat.shape[1])
            fv = take(n * C)
            out["feature"] = (fv if feat.dtype == t.float64 else fv.astype(np.int32).view(np.float32)).reshape(n, C)
        return out


_landing = {}


def _pinned_landing(numel):
    """Grow-only pinned fp64 host buffer per device for GridSampleResult reads."""
    t = nat.torch()
    dev = t.cuda.current_device()
    buf = _landing.get(dev)
    if buf is None or buf.numel() < numel:
        buf = _landing[dev] = t.empty(max(numel, 1 << 16), dtype=t.float64, pin_memory=True)
    return buf


_WS_BYTES = {}


def _grid_ws_bytes(npix):
    """xgs_grid_workspace, memoised (a pure function of the pixel count)."""
    b = _WS_BYTES.get(npix)
    if b is None:
        if len(_WS_BYTES) > 64:
            _WS_BYTES.clear()
        b = _WS_BYTES[npix] = int(nat.lib().xgs_grid_workspace(npix))
    return b


def _intr4(intr):
    if isinstance(intr, CameraIntrinsics) or hasattr(intr, "fx"):   # ours or semsplat.core's
        return float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
    fx, fy, cx, cy = (float(v) for v in intr)
    return fx, fy, cx, cy


def _poses(poses, F):
    """list[CameraPose] | (R [F,3,3], t [F,3]) -> device fp64 (R, t)."""
    t = nat.torch()
    def _is_pose(p):   # ours or semsplat.core.CameraPose
        return isinstance(p, CameraPose) or (hasattr(p, "rotation") and hasattr(p, "translation"))
    if _is_pose(poses):
        poses = [poses]
    if isinstance(poses, (list, tuple)) and poses and _is_pose(poses[0]):
        R = np.stack([p.rotation for p in poses])
        tr = np.stack([p.translation for p in poses])
    else:
        R, tr = poses
    R = R if is_tensor(R) else t.from_numpy(np.ascontiguousarray(np.asarray(R, dtype=np.float64)))
    tr = tr if is_tensor(tr) else t.from_numpy(np.ascontiguousarray(np.asarray(tr, dtype=np.float64)))
    R = R.to(device="cuda", dtype=t.float64).reshape(-1, 9).contiguous()
    tr = tr.to(device="cuda", dtype=t.float64).reshape(-1, 3).contiguous()
    if R.shape[0] != F or tr.shape[0] != F:
        raise InvalidInputError("one pose per frame required")
    return R, tr


def _dev(a, dtype):
    t = nat.torch()
    if a is None:
        return None
    if is_tensor(a):
        return a.to(device="cuda", dtype=dtype).contiguous()
    np_dt = {t.float32: np.float32, t.uint8: np.uint8}[dtype]
    return t.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np_dt))).to("cuda")


class GridSampler:
    """Incremental voxel grid sampler bound to one map (its occupancy set).

    ``sample`` processes a batch of frames; frames in a batch behave exactly
    like frames submitted one by one in order (first occurrence over
    (frame, pixel) wins, later frames see the earlier frames' voxels).
    """

    def __init__(self, intrinsics, voxel_size: float, stride: int = 1, mode: str = "first",
                 min_scale: float = 1e-3, occupied: Optional[VoxelHashSet] = None, capacity: int = 1 << 20):
        if voxel_size <= 0:
            raise InvalidInputError("voxel size must be positive")
        if stride < 1:
            raise InvalidInputError("stride must be >= 1")
        if mode not in ("first", "mean"):
            raise InvalidInputError("mode must be 'first' or 'mean'")
        self.intr = _intr4(intrinsics)
        self.voxel = float(voxel_size)
        self.stride = int(stride)
        self.mode = mode
        self.min_scale = float(min_scale)
        self.occupied = occupied if occupied is not None else VoxelHashSet(capacity)

    @staticmethod
    def _pinned(a, dtype):
        t = nat.torch()
        return (isinstance(a, t.Tensor) and a.device.type == "cpu" and a.is_pinned() and a.dtype == dtype
                and a.is_contiguous())

    def sample(self, depth, poses, color=None, features=None) -> GridSampleResult:
        t = nat.require_cuda()
        # pinned host frames go to the device inside the native call (frame
        # chunks copied while earlier frames' keys are computed)
        host = self._pinned(depth, t.float32) and (color is None or self._pinned(color, t.uint8))
        d = depth if host else _dev(depth, t.float32)
        if d.dim() == 2:
            d = d.unsqueeze(0)
        if d.dim() != 3:
            raise InvalidInputError("depth must be (H, W) or (F, H, W)")
        F, H, W = (int(v) for v in d.shape)
        R, tr = _poses(poses, F)
        col = color if host else _dev(color, t.uint8)
        if col is not None:
            col = col.reshape(F, H, W, 3) if col.dim() != 4 else col
            if tuple(col.shape) != (F, H, W, 3):
                raise InvalidInputError("color must be (F, H, W, 3) uint8")
        stage = None
        if host:   # grow-only device staging buffers
            key = (F, H, W, col is not None)
            stage = getattr(self, "_stage", None)
            if stage is None or stage[0] != key:
                stage = (key, t.empty((F, H, W), dtype=t.float32, device="cuda"),
                         t.empty((F, H, W, 3), dtype=t.uint8, device="cuda") if col is not None else None)
                self._stage = stage
        feat = _dev(features, t.float32) if features is not None else None
        if feat is not None:
            # (F, C, Hf, Wf): one map per frame (supervision.py:133-147 gather);
            # a single (C, Hf, Wf) map is accepted for a one-frame batch only
            if feat.dim() == 3 and F == 1:
                feat = feat.unsqueeze(0)
            if feat.dim() != 4 or int(feat.shape[0]) != F or min(int(v) for v in feat.shape[1:]) < 1:
                raise InvalidInputError(f"features must be (F={F}, C, Hf, Wf); got {tuple(feat.shape)}")
        s = self.stride
        cap = max(1, F * ((H + s - 1) // s) * ((W + s - 1) // s))
        C = int(feat.shape[1]) if feat is not None else 0
        # one fp64 allocation for every per-voxel field (key and pid as int64
        # views): [key | pid | mu x3 | color x3 | scale | depth | count]
        flat = t.empty(11 * cap, dtype=t.float64, device="cuda")
        # first-pick copies the gathered fp32 value; mean mode averages in fp64
        fdt = t.float32 if self.mode == "first" else t.float64
        ofeat = t.empty((cap, C), dtype=fdt, device="cuda") if feat is not None else None
        b = flat.data_ptr()
        fx, fy, cx, cy = self.intr
        fr = nat.GridFrames(F, H, W, d.data_ptr(), col.data_ptr() if col is not None else None, R.data_ptr(),
                            tr.data_ptr(), fx, fy, cx, cy, self.voxel, s, 0 if self.mode == "first" else 1,
                            self.min_scale, feat.data_ptr() if feat is not None else None,
                            C, int(feat.shape[2]) if feat is not None else 0,
                            int(feat.shape[3]) if feat is not None else 0)
        res = nat.GridResult(cap, b, b + 8 * cap, b + 16 * cap, b + 40 * cap, b + 64 * cap, b + 72 * cap,
                             ofeat.data_ptr() if ofeat is not None else None, b + 80 * cap, 0, 0, 0, 0, 0,
                             nat.F32 if fdt == t.float32 else nat.F64)
        ws = nat.workspace("grid", _grid_ws_bytes(F * H * W))
        if host:
            nat.call("xgs_grid_sample_h2d", ctypes.byref(fr), stage[1].data_ptr(),
                     stage[2].data_ptr() if stage[2] is not None else None, self.occupied._h, ctypes.byref(res),
                     nat.ptr(ws), ws.numel(), nat.stream_ptr())
        else:
            nat.call("xgs_grid_sample", ctypes.byref(fr), self.occupied._h, ctypes.byref(res), nat.ptr(ws),
                     ws.numel(), nat.stream_ptr())
        return GridSampleResult(flat, cap, int(res.n_new), ofeat, int(res.n_valid), int(res.n_voxels),
                                int(res.n_sorted), int(res.sort_passes))


class GridGraph:
    """A first-pick grid batch captured into a CUDA graph (xgs_grid_sample with
    XGS_GRID_ASYNC): :meth:`replay` re-runs the whole batch -- front end, table
    scan + map test, pid list, emit -- with one graph launch and no host sync,
    on the same device buffers (write the next batch into :attr:`depth`,
    :attr:`R`, :attr:`T`, :attr:`color`, :attr:`features`); :meth:`result`
    synchronises and returns it as a :class:`GridSampleResult`.

    Building it runs the given batch once synchronously through
    :meth:`GridSampler.sample` (that call sizes the library's per-device state
    the asynchronous call needs; its voxels enter the map as usual) and keeps
    that result as :attr:`first`.  The map must keep its capacity afterwards:
    the asynchronous call does not grow it (``VoxelHashSet`` sized for the
    stream, as PerceiverStream does)."""

    def __init__(self, sampler: "GridSampler", depth, poses, color=None, features=None):
        t = nat.require_cuda()
        if sampler.mode != "first":
            raise InvalidInputError("graph capture supports first-pick sampling only")
        self.sampler = sampler
        d = _dev(depth, t.float32)
        d = d.unsqueeze(0) if d.dim() == 2 else d
        F, H, W = (int(v) for v in d.shape)
        R, tr = _poses(poses, F)
        self.depth, self.R, self.T = d.clone(), R.clone(), tr.clone()
        self.color = _dev(color, t.uint8).reshape(F, H, W, 3).clone() if color is not None else None
        self.features = _dev(features, t.float32).clone() if features is not None else None
        self.first = sampler.sample(self.depth, (self.R, self.T), self.color, features=self.features)
        s = sampler.stride
        self.cap = cap = max(1, F * ((H + s - 1) // s) * ((W + s - 1) // s))
        C = int(self.features.shape[1]) if self.features is not None else 0
        self.flat = t.empty(11 * cap, dtype=t.float64, device="cuda")
        self.ofeat = t.empty((cap, C), dtype=t.float32, device="cuda") if C else None
        self.dev_status = t.zeros(4, dtype=t.int64, device="cuda")
        # the graph holds the workspace's address: owned by this object (freed with it)
        self.ws = t.empty(max(int(_grid_ws_bytes(F * H * W)), 256), dtype=t.uint8, device="cuda")
        fx, fy, cx, cy = sampler.intr
        ft = self.features
        self._fr = nat.GridFrames(F, H, W, self.depth.data_ptr(),
                                  self.color.data_ptr() if self.color is not None else None, self.R.data_ptr(),
                                  self.T.data_ptr(), fx, fy, cx, cy, sampler.voxel, s, 0, sampler.min_scale,
                                  ft.data_ptr() if ft is not None else None, C,
                                  int(ft.shape[2]) if ft is not None else 0, int(ft.shape[3]) if ft is not None else 0,
                                  nat.GRID_ASYNC)
        b = self.flat.data_ptr()
        self._res = nat.GridResult(cap, b, b + 8 * cap, b + 16 * cap, b + 40 * cap, b + 64 * cap, b + 72 * cap,
                                   self.ofeat.data_ptr() if self.ofeat is not None else None, b + 80 * cap, 0, 0, 0,
                                   0, 0, nat.F32, self.dev_status.data_ptr())
        g = t.cuda.CUDAGraph()
        st = t.cuda.Stream()
        st.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(st):
            with t.cuda.graph(g, stream=st):
                nat.call("xgs_grid_sample", ctypes.byref(self._fr), sampler.occupied._h, ctypes.byref(self._res),
                         nat.ptr(self.ws), self.ws.numel(), nat.stream_ptr())
        t.cuda.current_stream().wait_stream(st)
        self.graph = g

    def replay(self):
        """Enqueue the batch on the current stream (no host sync)."""
        self.graph.replay()

    def result(self) -> GridSampleResult:
        """Synchronise and return the last replayed batch (views of the graph's
        output buffers: valid until the next replay)."""
        n_new, n_valid, n_vox, err = (int(v) for v in self.dev_status.cpu())
        if err:
            raise InvalidStateError(f"grid batch overflow (code {err}): the map set or batch table is full")
        return GridSampleResult(self.flat, self.cap, n_new, self.ofeat, n_valid, n_vox)


def radix_sort_pairs(keys, vals, bits: int = 64):
    """In-house stable LSD radix sort of (uint64 key, uint32 value) pairs (CUDA tensors, in place)."""
    t = nat.require_cuda()
    n = int(keys.numel())
    ws = nat.workspace("sort", nat.lib().xgs_grid_workspace(n))
    nat.call("xgs_radix_sort_pairs_u64", nat.ptr(keys), nat.ptr(vals), n, int(bits), nat.ptr(ws), ws.numel(),
             nat.stream_ptr())
    return keys, vals
