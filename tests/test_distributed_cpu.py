"""Multi-GPU VQ host logic on CPU: world_size 2 over gloo.

DataParallelVQ (paper_2603_09632_b200/distributed.py) shards the rows, packs
[sums | counts] into one all-reduce, runs the EMA on every rank and revives
dead codes from a reservoir distributed over the ranks.  Here the device
backend is replaced by the CPU oracle (test-only backend) so the sharding,
packing, reservoir ownership and revival broadcast are checked against the
single-process reference semantics (oracle.vq.online_step on the concatenated
batch): counts / N bit-exact, sums / M / E within 1e-12 relative (the
all-reduce changes the partial-sum order), revived code lists identical.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import native as on
from oracle import vq as ov
from paper_2603_09632_b200.distributed import DataParallelVQ, ReservoirMap, strong_shard
from paper_2603_09632_b200.vq import VqConfig


class OracleBackend:
    """CPU stand-in for CudaBackend (state = (E, N, M) float64 tensors)."""

    def __init__(self, K, D, lam, eps):
        self.K, self.D, self.lam, self.eps = K, D, lam, eps

    def int_tensor(self, v):
        return torch.tensor(v, dtype=torch.int64)

    def prepare(self, shard):
        return torch.as_tensor(shard)

    def rows(self, shard):
        return int(shard.shape[0])

    def new_ring(self, cap):
        return np.zeros((cap, self.D))

    def ring_write(self, ring, shard, first, cnt, phys):
        x = shard.numpy()
        for j in range(cnt):
            ring[(phys + j) % ring.shape[0]] = x[first + j]

    def local_stats(self, state, shard, cfg):
        E = state[0].numpy()
        x = shard.numpy()
        packed = np.zeros(self.K * self.D + self.K)
        if x.shape[0]:
            codes = on.assign(x, E)
            counts, sums = on.accumulate(x, codes, self.K)
            packed[:self.K * self.D] = sums.reshape(-1)
            packed[self.K * self.D:] = counts
        return torch.from_numpy(packed)

    def ema(self, state, packed):
        p = packed.numpy()
        cb = ov.OracleCodebook(state[0].numpy(), state[1].numpy(), state[2].numpy(), self.lam, self.eps)
        out = ov.ema_step(cb, p[self.K * self.D:], p[:self.K * self.D].reshape(self.K, self.D))
        return (torch.from_numpy(out.E), torch.from_numpy(out.N), torch.from_numpy(out.M))

    def counts_host(self, state):
        return state[1].numpy()

    def gather_owned(self, ring, owners, rank):
        rows = torch.zeros((len(owners), self.D), dtype=torch.float64)
        for i, (r, phys) in enumerate(owners):
            if r == rank:
                rows[i] = torch.from_numpy(ring[phys])
        return rows

    def take(self, rows, idx):
        return rows[idx].contiguous()

    def put(self, rows, idx, buf):
        rows[idx] = buf
        return rows

    def revive(self, state, dead, rows):
        E, N, M = (s.clone() for s in state)
        for i, k in enumerate(dead):
            M[k] = rows[i]
            N[k] = 1.0 + self.eps
            E[k] = M[k] / (N[k] + self.eps)
        return (E, N, M)


def make_stream(seed, steps, n, K, D):
    rng = np.random.default_rng(seed)
    C = rng.normal(size=(6, D))
    E0 = np.concatenate([C[:3] + 0.01, rng.normal(size=(K - 3, D)) * 30.0])   # far codes die
    batches = [C[rng.integers(0, 6, n)] + 0.05 * rng.normal(size=(n, D)) for _ in range(steps)]
    return E0, batches


def worker(rank, world, port, out_path, sizes):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    K, D, steps = 8, 5, 12
    E0, batches = make_stream(3, steps, sum(sizes), K, D)
    cfg = VqConfig(K=K, lam=0.7, gamma=0.5 / K, delta_dead=1e-2, reservoir_capacity=150)
    be = OracleBackend(K, D, 0.7, 1e-5)
    vq = DataParallelVQ((torch.from_numpy(E0.copy()), torch.zeros(K, dtype=torch.float64),
                         torch.zeros(K, D, dtype=torch.float64)), cfg, np.random.default_rng(9), be)
    revived = []
    off = [0] + list(np.cumsum(sizes))
    for b in batches:
        shard = torch.from_numpy(b[off[rank]:off[rank + 1]].copy())
        rev, _ = vq.step(shard, sizes)
        revived.append(rev)
    if rank == 0:
        np.savez(out_path, E=vq.state[0].numpy(), N=vq.state[1].numpy(), M=vq.state[2].numpy(),
                 revived=np.array([len(r) for r in revived]), rlist=np.concatenate([np.array(r, dtype=int)
                                                                                     for r in revived] + [[]]))
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("sizes", [(100, 100), (30, 170), tuple(strong_shard(200, 4, r)[1] for r in range(4))])
def test_multi_rank_vq_matches_single_process(tmp_path, sizes):
    """A FIXED global batch split across the ranks (strong scaling, as the
    bench's C5 mode shards 67,108,864 rows / N) gives the single-process
    online_step result."""
    out = str(tmp_path / "r.npz")
    world = len(sizes)
    mp.start_processes(worker, args=(world, free_port(), out, sizes), nprocs=world, join=True, start_method="spawn")
    got = np.load(out)
    K, D, steps = 8, 5, 12
    E0, batches = make_stream(3, steps, sum(sizes), K, D)
    cb = ov.OracleCodebook(E0.copy(), np.zeros(K), np.zeros((K, D)), 0.7, 1e-5, ov.OracleReservoir(150, D))
    rng = np.random.default_rng(9)
    revived = []
    for b in batches:
        cb, rev, _ = ov.online_step(cb, b, 0.7, 0.5 / K, 1e-2, rng, assume_all_pass=True)
        revived.append(rev)
    assert sum(len(r) for r in revived) > 0        # the stream exercises revival
    assert list(got["revived"]) == [len(r) for r in revived]
    assert np.array_equal(got["N"], cb.N)
    np.testing.assert_allclose(got["M"], cb.M, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(got["E"], cb.E, rtol=1e-12, atol=1e-13)


def test_strong_shard_tiles_the_batch():
    for total, world in ((67_108_864, 1), (67_108_864, 2), (67_108_864, 8), (1000, 3), (7, 8)):
        parts = [strong_shard(total, world, r) for r in range(world)]
        assert parts[0][0] == 0 and sum(n for _, n in parts) == total
        for (f0, n0), (f1, _) in zip(parts, parts[1:]):
            assert f1 == f0 + n0
        assert max(n for _, n in parts) - min(n for _, n in parts) <= 1
    assert strong_shard(67_108_864, 8, 3) == (3 * 8_388_608, 8_388_608)
    with pytest.raises(ValueError):
        strong_shard(10, 2, 2)


def test_reservoir_map_ownership():
    rm = ReservoirMap(capacity=10, world=3)
    rm.add_step([4, 0, 3])        # global rows 0..6: r0 0-3, r2 4-6
    assert len(rm) == 7
    assert rm.locate(0) == (0, 0) and rm.locate(4) == (2, 0) and rm.locate(6) == (2, 2)
    assert rm.ring_writes(2, 3) == (0, 3, 0)
    rm.add_step([5, 5, 5])        # global rows 7..21 -> reservoir = rows 12..21
    assert len(rm) == 10
    # logical 0 = global 12 = rank 1's first row of this step (own index 0)
    assert rm.locate(0) == (1, 0)
    assert rm.locate(9) == (2, (3 + 4) % 10)
    assert rm.ring_writes(0, 5) == (0, 5, 4)
    rm.add_step([0, 0, 25])       # a shard larger than the capacity
    assert rm.ring_writes(2, 25) == (15, 10, (8 + 15) % 10)
    assert all(rm.locate(i)[0] == 2 for i in range(10))
