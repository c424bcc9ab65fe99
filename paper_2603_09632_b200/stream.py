"""Per-frame Perceiver step as ONE CUDA graph (BASELINE configs[3], C4).

The reference's per-keyframe path is: new Gaussians from the RGB-D frame
(``slam.densify_and_prune``'s insertion, slam.py:601-651, here the voxel
sampler of grid.py) whose semantic features then feed ``vq.online_step``
(vq.py:193-212).  At ~2K new points per 640x480 frame the work is a few
microseconds of kernels, so the per-frame latency is set by launches and
host round trips.  ``PerceiverStream`` therefore captures the device part
once and replays it per frame over fixed-capacity buffers:

  graph:  grid sampling (xgs_grid_sample, XGS_GRID_ASYNC: no host sync) of the
          staged frame -> new voxels in pixel order + their features gathered
          from the frame's feature map (supervision.py:133-147 rule)
          -> valid-row mask of the first n_new rows (xgs_prefix_mask; n_new
          lives on the device) -> assign (tcgen05 screen + exact re-rank) of
          the first min(n_new, `vq_capacity`) rows of the feature window
          (xgs_vq_assign_dev) -> masked accumulate (counting sort + sequential
          fp64 chains; rows past n_new contribute nothing, so the statistics
          equal the reference's on the n_new rows) -> EMA into the other of two
          codebook states -> reservoir append of the n_new rows (vq.py:203,
          xgs_vq_ring_write_dev: row count and ring position on the device).
  host:   ONE device->host read of {N (K fp64), n_new, n_valid, n_voxels,
          error} -> the FIFO bookkeeping of the append -> the reference's host
          RNG draws for dead codes -> revival kernel.

Two graphs alternate between the two codebook states (graph i reads state i,
writes state 1 - i), so a frame whose VQ step must not apply keeps the
current state: a frame without new points, or one with more than
`vq_capacity` -- rare at C4, its VQ would have seen only the window -- which is
redone through the synchronous ``online_step`` on exactly its n_new rows.
Results are bit-identical to ``GridSampler.sample(...)`` followed by
``online_step`` on the returned features, reservoir included
(tests/test_stream_gpu.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .core import Codebook, FeatureReservoir
from .errors import InvalidInputError
from .grid import GridSampler, VoxelHashSet, _grid_ws_bytes, _intr4


@dataclass
class StreamStepResult:
    n_new: int            # new Gaussians (voxels) of the frame
    n_valid: int          # valid depth pixels
    n_voxels: int         # distinct voxels of the frame (new or already mapped)
    revived: list         # dead codes revived this step (vq.py:173-190)
    graph: bool           # served by the graph replay (False: synchronous fallback)


class PerceiverStream:
    """Grid sampling -> online VQ per frame, device part replayed as a CUDA graph."""

    def __init__(self, intrinsics, height: int, width: int, voxel_size: float, codebook: Codebook, cfg,
                 feat_shape, rng: np.random.Generator, map_capacity: int = 1 << 23, vq_capacity: int = 16384,
                 min_scale: float = 1e-3):
        t = nat.require_cuda()
        if not codebook.on_device:
            codebook = codebook.to_device()
        C, Hf, Wf = (int(v) for v in feat_shape)
        if C != codebook.D:
            raise InvalidInputError(f"feature channels {C} != codebook D={codebook.D}")
        self.t, self.cfg, self.rng = t, cfg, rng
        self.H, self.W, self.C = int(height), int(width), C
        self.K, self.D = codebook.K, codebook.D
        self.lam, self.eps = float(codebook.lam), float(codebook.epsilon)
        self.intr = _intr4(intrinsics)
        self.voxel = float(voxel_size)
        self.min_scale = float(min_scale)
        dev = "cuda"
        # codebook state, double-buffered: graph i reads state i and writes the EMA
        # into state 1 - i, so a frame whose VQ step must not apply (no new points,
        # or more than the window) simply keeps the current state -- no snapshot
        # copies per frame.  The revival and the host fallback update the current one.
        E = codebook.E.clone().contiguous()
        N = codebook.N.clone().contiguous()
        M = codebook.M.clone().contiguous()
        self._S = [(E, N, M), (t.empty_like(E), t.empty_like(N), t.empty_like(M))]
        self._cur = 0
        self.reservoir = codebook.reservoir if codebook.reservoir is not None else FeatureReservoir(
            cfg.reservoir_capacity, self.D)
        # staged frame (the graph reads these addresses)
        self.depth = t.zeros((1, self.H, self.W), dtype=t.float32, device=dev)
        self.color = t.zeros((1, self.H, self.W, 3), dtype=t.uint8, device=dev)
        self.R = t.zeros((1, 9), dtype=t.float64, device=dev)
        self.T = t.zeros((1, 3), dtype=t.float64, device=dev)
        self.feat = t.zeros((1, C, Hf, Wf), dtype=t.float32, device=dev)
        # fixed-capacity outputs (every pixel could be a new voxel)
        self.cap = self.H * self.W
        self.flat = t.zeros(11 * self.cap, dtype=t.float64, device=dev)
        self.ofeat = t.zeros((self.cap, C), dtype=t.float32, device=dev)
        self.vcap = min(int(vq_capacity), self.cap)
        self.mask = t.zeros(self.vcap, dtype=t.uint8, device=dev)
        self.codes = t.zeros(self.vcap, dtype=t.int64, device=dev)
        self.packed = t.zeros(self.K * self.D + self.K, dtype=t.float64, device=dev)
        self.dev_status = t.zeros(4, dtype=t.int64, device=dev)
        # the reservoir ring's next write row on the device (the graph appends the
        # frame's new rows there; the host mirrors the FIFO after reading n_new)
        self.reservoir._ensure()
        self.ring_start = t.zeros(1, dtype=t.int64, device=dev)
        self.host_N = t.empty(self.K, dtype=t.float64, pin_memory=True)
        self.host_status = t.empty(4, dtype=t.int64, pin_memory=True)
        self._host_N_np, self._host_status_np = self.host_N.numpy(), self.host_status.numpy()   # views, made once
        self.occupied = VoxelHashSet(map_capacity)
        self.sampler = GridSampler(intrinsics, voxel_size, occupied=self.occupied, min_scale=min_scale)
        # the graph holds the workspaces' addresses: owned by this stream (a shared,
        # grow-only library workspace could be reallocated under the graph)
        L = nat.lib()
        ws = lambda n: t.empty(max(int(n), 256), dtype=t.uint8, device=dev)
        self.ws_grid = ws(_grid_ws_bytes(self.cap))
        self.ws_assign = ws(L.xgs_vq_assign_workspace(self.vcap, self.K, C, nat.F32, C))
        self.ws_acc = ws(L.xgs_vq_accumulate_workspace(self.vcap, self.K))
        fx, fy, cx, cy = self.intr
        self._frames = nat.GridFrames(1, self.H, self.W, self.depth.data_ptr(), self.color.data_ptr(),
                                      self.R.data_ptr(), self.T.data_ptr(), fx, fy, cx, cy, self.voxel, 1, 0,
                                      self.min_scale, self.feat.data_ptr(), C, Hf, Wf, nat.GRID_ASYNC)
        b, c = self.flat.data_ptr(), self.cap
        self._result = nat.GridResult(c, b, b + 8 * c, b + 16 * c, b + 40 * c, b + 64 * c, b + 72 * c,
                                      self.ofeat.data_ptr(), b + 80 * c, 0, 0, 0, 0, 0, nat.F32,
                                      self.dev_status.data_ptr())
        # rows past n_new in the assign window hold stale finite features; start
        # them as a real codeword (a unique nearest code: no re-rank work)
        self.ofeat[:self.vcap].copy_(self.E[0].to(t.float32).expand(self.vcap, C))
        self.graph = None
        self.frames = 0

    E = property(lambda self: self._S[self._cur][0])
    N = property(lambda self: self._S[self._cur][1])
    M = property(lambda self: self._S[self._cur][2])

    # ------------------------------------------------------------ device part
    def _enqueue(self, i):
        """Graph i's body (all on the current stream, no host sync): state i in,
        the EMA into state 1 - i."""
        t, L, sp = self.t, nat.lib(), nat.stream_ptr()
        Ei, Ni, Mi = self._S[i]
        Eo, No, Mo = self._S[1 - i]
        nat.check(L.xgs_grid_sample(ctypes.byref(self._frames), self.occupied._h, ctypes.byref(self._result),
                                    nat.ptr(self.ws_grid), self.ws_grid.numel(), sp))
        nat.check(L.xgs_prefix_mask(nat.ptr(self.dev_status), self.vcap, nat.ptr(self.mask), sp))
        # only the frame's new rows (the count the grid batch wrote on the device)
        nat.check(L.xgs_vq_assign_dev(nat.ptr(self.ofeat), nat.F32, self.vcap, self.C, self.C, nat.ptr(Ei), self.K,
                                      nat.ptr(self.codes), nat.ptr(self.ws_assign), self.ws_assign.numel(),
                                      nat.ptr(self.dev_status), sp))
        sums = self.packed[:self.K * self.D]
        counts = self.packed[self.K * self.D:]
        nat.check(L.xgs_vq_accumulate(nat.ptr(self.ofeat), nat.F32, self.vcap, self.C, self.C, nat.ptr(self.codes),
                                      nat.ptr(self.mask), self.K, nat.ptr(counts), nat.ptr(sums),
                                      nat.ptr(self.ws_acc), self.ws_acc.numel(), sp))
        nat.check(L.xgs_vq_ema(self.lam, self.eps, self.K, self.D, nat.ptr(Ni), nat.ptr(Mi),
                               nat.ptr(counts), nat.ptr(sums), nat.ptr(No), nat.ptr(Mo), nat.ptr(Eo), sp))
        # reservoir extend of the frame's new rows (vq.py:203; rows past vcap are the
        # host fallback's, which rewinds the position first)
        res = self.reservoir
        nat.check(L.xgs_vq_ring_write_dev(nat.ptr(self.ofeat), nat.F32, self.C, nat.ptr(self.dev_status), self.vcap,
                                          self.C, nat.ptr(res._ring), res.capacity, nat.ptr(self.ring_start), sp))
        self.host_N.copy_(No, non_blocking=True)
        self.host_status.copy_(self.dev_status, non_blocking=True)

    def _sync_ring_start(self):
        self.ring_start.fill_(self.reservoir._write_pos())

    def _capture(self):
        t = self.t
        self._sync_ring_start()
        graphs = []
        for i in (0, 1):
            g = t.cuda.CUDAGraph()
            s = t.cuda.Stream()
            s.wait_stream(t.cuda.current_stream())
            with t.cuda.stream(s):
                with t.cuda.graph(g, stream=s):
                    self._enqueue(i)
            t.cuda.current_stream().wait_stream(s)
            graphs.append(g)
        self.graphs = graphs
        self.graph = graphs[0]

    # ------------------------------------------------------------ per frame
    def inputs(self):
        """The staging tensors the graph reads: (depth (1, H, W) fp32, R (1, 9)
        fp64, t (1, 3) fp64, colour (1, H, W, 3) u8, features (1, C, Hf, Wf)
        fp32).  A producer that writes the next frame into them directly
        saves step() the staging copies."""
        return self.depth, self.R, self.T, self.color, self.feat

    def _stage(self, depth, R, T, color, feats):
        for dst, src in ((self.depth, depth), (self.color, color), (self.R, R), (self.T, T), (self.feat, feats)):
            if src.data_ptr() != dst.data_ptr():
                dst.view(-1).copy_(src.reshape(-1), non_blocking=True)

    def _sync_frame(self):
        """Synchronous path on the staged frame (first frame: sizes the library
        state the async call needs)."""
        from .vq import online_step
        r = self.sampler.sample(self.depth, (self.R, self.T), self.color, features=self.feat)
        cb = Codebook._make(self.E, self.N, self.M, self.lam, self.eps, self.reservoir)
        if len(r):
            cb, res = online_step(cb, r.feature, self.cfg, self.rng)
            self.E.copy_(cb.E)
            self.N.copy_(cb.N)
            self.M.copy_(cb.M)
            revived = res.revived
        else:
            revived = []
        self.t.cuda.current_stream().synchronize()
        return StreamStepResult(len(r), r.n_valid, r.n_voxels, revived, False)

    def step(self, depth, pose, color, feats) -> StreamStepResult:
        """One frame: depth (H, W) fp32, pose (R (3, 3), t (3,)) fp64, colour
        (H, W, 3) uint8, features (C, Hf, Wf) fp32 -- CUDA tensors."""
        from .vq import _revive_dev, online_step
        R, T = pose
        self._stage(depth, R, T, color, feats)
        self.frames += 1
        if self.graph is None:
            out = self._sync_frame()
            self._capture()
            return out
        self.graphs[self._cur].replay()
        self.t.cuda.current_stream().synchronize()
        n_new, n_valid, n_vox, err = self._host_status_np.tolist()
        if err:
            raise RuntimeError(f"grid batch overflow (code {err}): the map set or batch table is full")
        if n_new == 0:          # no new points: the stream makes no VQ step (online_step needs a nonempty batch)
            return StreamStepResult(0, n_valid, n_vox, [], True)   # (the current state is untouched)
        if n_new > self.vcap:   # the window missed rows: redo the VQ on all n_new rows from the current state
            cb = Codebook._make(self.E, self.N, self.M, self.lam, self.eps, self.reservoir)
            # (its reservoir extend rewrites, from the same position, the vcap rows the
            # graph appended; the host FIFO was not advanced for them)
            cb, res = online_step(cb, self.ofeat[:n_new], self.cfg, self.rng)
            self.E.copy_(cb.E)
            self.N.copy_(cb.N)
            self.M.copy_(cb.M)
            self._sync_ring_start()
            self.t.cuda.current_stream().synchronize()
            return StreamStepResult(n_new, n_valid, n_vox, res.revived, False)
        self._cur = 1 - self._cur   # the EMA'd state becomes current
        revived = []
        if n_new:
            # the graph appended the batch to the reservoir ring (vq.py:203): mirror
            # the FIFO, then the host RNG revival
            self.reservoir._account(n_new)
            cb = Codebook._make(self.E, self.N, self.M, self.lam, self.eps, self.reservoir)
            revived, _ = _revive_dev(cb, self.E, self.N, self.M, self.cfg.delta_dead, self.rng,
                                     N_host=self._host_N_np)
        return StreamStepResult(n_new, n_valid, n_vox, revived, True)

    def codebook(self) -> Codebook:
        return Codebook._make(self.E, self.N, self.M, self.lam, self.eps, self.reservoir)

    def new_voxels(self, n):
        """The last frame's first n new voxels (key, pid, mu, colour, scale, depth, count, feature)."""
        from .grid import GridSampleResult
        return GridSampleResult(self.flat, self.cap, int(n), self.ofeat, -1, -1)
