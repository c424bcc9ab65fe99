"""The real multi-rank VQ code path (DataParallelVQ + CudaBackend, libxgs
kernels) with world_size 2, both ranks on cuda:0, collectives over gloo (host
mediated, no device-side waits).  Result vs the single-process GPU run on the
concatenated batch: N bit-exact, M / E within 1e-12 relative."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

K, D, STEPS, SIZES = 64, 96, 6, (700, 1300)


def stream():
    rng = np.random.default_rng(8)
    C = rng.normal(size=(80, D))
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    n = sum(SIZES)
    batches = []
    for _ in range(STEPS):
        x = C[rng.integers(0, 70, n)] + 0.1 * rng.normal(size=(n, D))
        batches.append((x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32))
    E0 = np.concatenate([C[:K - 8] + 0.01, rng.normal(size=(8, D)) * 20]).astype(np.float64)  # 8 die
    return E0, batches


def run(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
    from paper_2603_09632_b200.vq import VqConfig
    E0, batches = stream()
    cfg = VqConfig(K=K, lam=0.9, gamma=0.5 / K, delta_dead=1e-2, reservoir_capacity=1000)
    vq = DataParallelVQ((torch.from_numpy(E0).cuda(), torch.zeros(K, dtype=torch.float64, device="cuda"),
                         torch.zeros(K, D, dtype=torch.float64, device="cuda")), cfg, np.random.default_rng(5),
                        CudaBackend(K, D, 0.9, 1e-5))
    off = [0, SIZES[0], sum(SIZES)] if world > 1 else [0, sum(SIZES)]
    revived = []
    for b in batches:
        sh = torch.from_numpy(b[off[rank]:off[rank + 1]]).cuda()
        rev, _ = vq.step(sh, list(SIZES) if world > 1 else [sum(SIZES)])
        revived.append(len(rev))
    if rank == 0:
        np.savez(out, E=vq.state[0].cpu().numpy(), N=vq.state[1].cpu().numpy(), M=vq.state[2].cpu().numpy(),
                 rev=np.array(revived))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_match_single(tmp_path, cuda):
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    single, multi = str(tmp_path / "s.npz"), str(tmp_path / "m.npz")
    run(0, 1, port, single)
    mp.start_processes(run, args=(2, port, multi), nprocs=2, join=True, start_method="spawn")
    a, b = np.load(single), np.load(multi)
    assert a["rev"].sum() > 0 and np.array_equal(a["rev"], b["rev"])
    assert np.array_equal(a["N"], b["N"])
    np.testing.assert_allclose(b["M"], a["M"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(b["E"], a["E"], rtol=1e-12, atol=1e-14)


def test_dataparallel_world1_matches_online_step(tmp_path, cuda):
    """DataParallelVQ (world 1) == the drop-in online_step, bit-exact, with revival."""
    import torch
    import paper_2603_09632_b200 as xv
    single = str(tmp_path / "s.npz")
    run(0, 1, 0, single)
    a = np.load(single)
    E0, batches = stream()
    cb = xv.Codebook(E=torch.from_numpy(E0).cuda(), N=torch.zeros(K, dtype=torch.float64, device="cuda"),
                     M=torch.zeros(K, D, dtype=torch.float64, device="cuda"), lam=0.9, epsilon=1e-5,
                     reservoir=xv.FeatureReservoir(1000, D))
    cfg = xv.VqConfig(K=K, lam=0.9, gamma=0.5 / K, delta_dead=1e-2, reservoir_capacity=1000)
    rng = np.random.default_rng(5)
    revived = []
    for b in batches:
        cb, res = xv.online_step(cb, torch.from_numpy(b).cuda(), cfg, rng)
        revived.append(len(res.revived))
    assert list(a["rev"]) == revived
    assert np.array_equal(a["N"], cb.N.cpu().numpy()) and np.array_equal(a["E"], cb.E.cpu().numpy())
