"""Data-parallel online VQ across the GPUs of one node.

Rows are sharded contiguously: rank r holds rows [off_r, off_r + n_r) of every
step's global batch (the global batch is the concatenation of the shards in
rank order).  One ``step`` is the reference's ``online_step`` (vq.py:193-212)
on that global batch:

  1. local assign + accumulate (libxgs kernels) on the shard;
  2. ONE all-reduce(sum) of the packed fp64 buffer [sums (K*D) | counts (K)]
     over NCCL/NVLink — the only data-path exchange;
  3. EMA on every rank (identical inputs -> identical codebooks);
  4. dead-code revival: every rank draws the same reservoir indices from the
     same host RNG; the reservoir is distributed — each rank keeps the last
     ``capacity`` rows of its own shard stream in a device ring, and a global
     reservoir index is mapped to (owner rank, ring row).  Only the drawn rows
     travel, broadcast from their owner.

With world_size == 1 the collectives vanish and the result is bit-identical to
the single-GPU ``online_step``.  Across ranks the partial-sum order differs, so
sums/E agree with the reference to ~1e-15 relative (not bitwise).

The local compute sits behind a small backend interface so the host logic
(sharding, packing, reservoir ownership, revival broadcast) is testable on CPU
with the gloo backend (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class _Segment:
    rank: int
    gstart: int      # global stream position of the first row
    n: int
    own_start: int   # index of the first row in the owner's own stream


class ReservoirMap:
    """Host bookkeeping of the distributed FIFO reservoir (core.py:178-203).

    The global reservoir is the last ``capacity`` rows of the global stream;
    every rank holds the same map and can resolve a logical reservoir index to
    (owner rank, physical ring row) without communication."""

    def __init__(self, capacity: int, world: int):
        self.capacity = int(capacity)
        self.world = int(world)
        self.total = 0                    # global rows seen
        self.own_total = [0] * world      # rows seen per rank
        self.segments: list[_Segment] = []

    def __len__(self):
        return min(self.capacity, self.total)

    def add_step(self, sizes):
        """Register one global batch made of per-rank shard sizes (rank order)."""
        g = self.total
        for r, n in enumerate(sizes):
            if n:
                self.segments.append(_Segment(r, g, int(n), self.own_total[r]))
                self.own_total[r] += int(n)
                g += int(n)
        self.total = g
        lo = self.total - len(self)
        self.segments = [s for s in self.segments if s.gstart + s.n > lo]

    def locate(self, i: int):
        """Logical reservoir index -> (rank, physical ring row of that rank)."""
        g = self.total - len(self) + int(i)
        for s in self.segments:
            if s.gstart <= g < s.gstart + s.n:
                return s.rank, (s.own_start + (g - s.gstart)) % self.capacity
        raise IndexError(i)

    def ring_writes(self, rank: int, n: int):
        """Where rank ``rank`` writes the last min(n, cap) rows of its new shard:
        (first shard row to copy, count, physical ring start)."""
        cap = self.capacity
        own0 = self.own_total[rank] - n   # own index of the shard's first row (after add_step)
        cnt = min(n, cap)
        first = n - cnt
        return first, cnt, (own0 + first) % cap


def strong_shard(total: int, world: int, rank: int):
    """Strong scaling (BASELINE configs[4]): the fixed global
    batch of ``total`` rows split into contiguous shards in rank order, the
    first ``total % world`` ranks taking one row more.  Returns (first global
    row, rows) of ``rank``; the shards tile [0, total) exactly."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard request")
    base, extra = divmod(int(total), int(world))
    rows = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    return first, rows


class DataParallelVQ:
    """Online VQ over row shards; ``backend`` does the device work."""

    def __init__(self, codebook_state, cfg, rng, backend, group=None):
        import torch.distributed as dist
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.group = group
        self.rank = self.dist.get_rank(group) if self.dist else 0
        self.world = self.dist.get_world_size(group) if self.dist else 1
        self.state = codebook_state          # backend-specific (E, N, M on device)
        self.cfg = cfg
        self.rng = rng
        self.be = backend
        self.res = ReservoirMap(cfg.reservoir_capacity, self.world)
        self.ring = backend.new_ring(cfg.reservoir_capacity)
        E, N, M = codebook_state
        K, D = getattr(backend, "K", None), getattr(backend, "D", None)
        if (tuple(E.shape) != (K, D) or tuple(M.shape) != (K, D) or tuple(N.shape) != (K,)):
            from .errors import InvalidInputError
            raise InvalidInputError(f"codebook state shapes {tuple(E.shape)}, {tuple(N.shape)}, {tuple(M.shape)} "
                                    f"do not match K={K}, D={D}")

    def _sizes(self, n_local):
        if self.world == 1:
            return [n_local]
        t = self.be.int_tensor([n_local])
        out = [self.be.int_tensor([0]) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [int(o.item()) for o in out]

    def step(self, shard, sizes=None):
        """One online_step on the global batch; returns the revived code list."""
        shard = self.be.prepare(shard)
        n_local = self.be.rows(shard)
        sizes = list(sizes) if sizes is not None else self._sizes(n_local)
        if sum(sizes) == 0:
            from .errors import InvalidInputError
            raise InvalidInputError("batch must be nonempty")
        # local statistics first (the device's long pole), one packed all-reduce
        packed = self.be.local_stats(self.state, shard, self.cfg)   # [sums | counts] fp64
        # reservoir (vq.py:203: extended before the mask/accumulate; the ring is
        # not read by the statistics, so enqueueing it second changes nothing):
        # every rank writes the tail of its shard
        self.res.add_step(sizes)
        first, cnt, phys = self.res.ring_writes(self.rank, n_local)
        if cnt:
            self.be.ring_write(self.ring, shard, first, cnt, phys)
        if self.world > 1:
            self.dist.all_reduce(packed, group=self.group)
        self.state = self.be.ema(self.state, packed)
        # revival with the shared host RNG (vq.py:173-190)
        N_host = self.be.counts_host(self.state)
        dead = np.nonzero(N_host < self.cfg.delta_dead)[0]
        if dead.size == 0 or len(self.res) == 0:
            return [], bool(dead.size)
        owners = [self.res.locate(int(self.rng.integers(0, len(self.res)))) for _ in dead]
        rows = self.be.gather_owned(self.ring, owners, self.rank)
        if self.world > 1:
            for r in sorted({o[0] for o in owners}):
                idx = [i for i, o in enumerate(owners) if o[0] == r]
                buf = self.be.take(rows, idx)
                self.dist.broadcast(buf, src=r, group=self.group)
                rows = self.be.put(rows, idx, buf)
        self.state = self.be.revive(self.state, dead, rows)
        return [int(k) for k in dead], False


class CudaBackend:
    """libxgs kernels on the current CUDA device (state = (E, N, M) tensors)."""

    def __init__(self, K, D, lam, eps):
        from . import _native as nat
        self.nat = nat
        self.t = nat.require_cuda()
        self._h2d, self._pending_host, self._packed = {}, None, None
        self.K, self.D, self.lam, self.eps = K, D, lam, eps

    def int_tensor(self, v):
        return self.t.tensor(v, dtype=self.t.int64, device="cuda")

    def rows(self, shard):
        return int(shard.shape[0])

    def prepare(self, shard):
        """Device rows as they are; pinned host rows get a (cached) device buffer
        that the statistics call fills chunk by chunk (H2D overlapped with the
        device work), see local_stats."""
        t = self.t
        if isinstance(shard, t.Tensor) and shard.device.type == "cpu" and shard.is_pinned() and shard.dim() == 2 \
                and shard.is_contiguous() and shard.dtype in (t.float32, t.float64, t.bfloat16):
            key = (tuple(shard.shape), shard.dtype)
            buf = self._h2d.get(key)
            if buf is None:
                self._h2d = {key: t.empty(shard.shape, dtype=shard.dtype, device="cuda")}
                buf = self._h2d[key]
            self._pending_host = shard
            return buf
        from .vq import _rows
        self._pending_host = None
        return _rows(shard)[0]

    def new_ring(self, cap):
        return self.t.empty((cap, self.D), dtype=self.t.float64, device="cuda")

    def ring_write(self, ring, shard, first, cnt, phys):
        from .vq import _rows
        xt, dt, n, d, ldx = _rows(shard)
        nat = self.nat
        nat.call("xgs_vq_ring_write", nat.ptr(xt), dt, ldx, first, cnt, d, nat.ptr(ring), ring.shape[0], phys,
                 nat.stream_ptr())

    def local_stats(self, state, shard, cfg):
        from .vq import _assign_accumulate_dev, _exact_dev, _rows, all_pass_provable
        t, nat = self.t, self.nat
        E = state[0]
        # the packed [sums | counts] buffer is consumed by the EMA (and the
        # all-reduce) on the same stream before the next step rewrites it
        packed = self._packed
        if packed is None or packed.device != E.device:
            packed = self._packed = t.empty(self.K * self.D + self.K, dtype=t.float64, device=E.device)
        sums = packed[:self.K * self.D].view(self.K, self.D)
        counts = packed[self.K * self.D:]
        n = self.rows(shard)
        if n == 0:
            packed.zero_()
            return packed
        host = getattr(self, "_pending_host", None)
        self._pending_host = None
        if host is not None and not all_pass_provable(cfg.gamma, self.K):
            shard.copy_(host)          # the exact confidence path needs the whole batch first
            host = None
        xt, dt, n, d, ldx = _rows(shard)
        if all_pass_provable(cfg.gamma, self.K):
            _assign_accumulate_dev(xt, dt, n, d, ldx, E, self.K, counts=counts, sums=sums, x_host=host)
            return packed
        else:
            _, _, codes, mask = _exact_dev(xt, dt, n, d, ldx, E, self.K, nat.EX_CODE | nat.EX_MASK,
                                           tau=cfg.tau_warm, gamma=cfg.gamma)
        ws = nat.workspace("accumulate", nat.lib().xgs_vq_accumulate_workspace(n, self.K))
        nat.call("xgs_vq_accumulate", nat.ptr(xt), dt, n, d, ldx, nat.ptr(codes), nat.ptr(mask), self.K,
                 nat.ptr(counts), nat.ptr(sums), nat.ptr(ws), ws.numel(), nat.stream_ptr())
        return packed

    def ema(self, state, packed):
        t, nat = self.t, self.nat
        E, N, M = state
        sums = packed[:self.K * self.D]
        counts = packed[self.K * self.D:]
        N2, M2, E2 = t.empty_like(N), t.empty_like(M), t.empty_like(E)
        nat.call("xgs_vq_ema", float(self.lam), float(self.eps), self.K, self.D, nat.ptr(N), nat.ptr(M),
                 nat.ptr(counts), nat.ptr(sums), nat.ptr(N2), nat.ptr(M2), nat.ptr(E2), nat.stream_ptr())
        return (E2, N2, M2)

    def counts_host(self, state):
        return state[1].cpu().numpy()

    def gather_owned(self, ring, owners, rank):
        t, nat = self.t, self.nat
        rows = t.zeros((len(owners), self.D), dtype=t.float64, device="cuda")
        mine = [i for i, o in enumerate(owners) if o[0] == rank]
        if mine:
            src = t.tensor([owners[i][1] for i in mine], dtype=t.int64, device="cuda")
            buf = t.empty((len(mine), self.D), dtype=t.float64, device="cuda")
            nat.call("xgs_gather_rows_f64", nat.ptr(ring), self.D, nat.ptr(src), len(mine), nat.ptr(buf),
                     nat.stream_ptr())
            rows[mine] = buf
        return rows

    def take(self, rows, idx):
        return rows[idx].contiguous()

    def put(self, rows, idx, buf):
        rows[idx] = buf
        return rows

    def revive(self, state, dead, rows):
        t, nat = self.t, self.nat
        E, N, M = state
        dk = t.from_numpy(np.asarray(dead, dtype=np.int64)).to("cuda")
        rr = t.arange(len(dead), dtype=t.int64, device="cuda")
        rows = rows.contiguous()
        nat.call("xgs_vq_revive", self.K, self.D, float(self.eps), nat.ptr(rows), rows.shape[0], nat.ptr(dk),
                 nat.ptr(rr), len(dead), nat.ptr(N), nat.ptr(M), nat.ptr(E), nat.stream_ptr())
        return (E, N, M)
