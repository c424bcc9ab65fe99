"""Bounded screening workspace: with the per-row screening buffers sized for
one row chunk (slot ring of two), a batch screened in many chunks must give
the same codes / counts / sums / codebook, bit for bit, as one chunk.  The
chunk size is forced small (XGS_SCREEN_CHUNK_ROWS=4096, read once at library
load) in a subprocess; the parent runs the default (single chunk)."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2603_09632_b200 as xv
from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
out = {}
for name, n, d, k, bf in (("f32", 50000, 128, 512, False), ("big", 30000, 96, 2048, False), ("bf16", 40000, 160, 512, True)):
    g = torch.Generator(device="cuda"); g.manual_seed(7)
    C = torch.randn(64, d, generator=g, device="cuda"); C /= C.norm(dim=1, keepdim=True)
    x = C[torch.randint(0, 64, (n,), generator=g, device="cuda")] + 0.1 * torch.randn(n, d, generator=g, device="cuda")
    x = x / x.norm(dim=1, keepdim=True)
    if bf:
        x = x.to(torch.bfloat16)
    E0 = x[torch.randint(0, n, (k,), generator=g, device="cuda")].double()
    cb = xv.Codebook._make(E0, torch.zeros(k, dtype=torch.float64, device="cuda"),
                           torch.zeros(k, d, dtype=torch.float64, device="cuda"), 0.99, 1e-5, None)
    out[name + "_codes"] = xv.assign_batch(x, cb).cpu().numpy()
    cfg = xv.VqConfig(K=k, lam=0.99, gamma=0.5 / k, delta_dead=1e-3)
    vq = DataParallelVQ((E0.clone(), torch.zeros(k, dtype=torch.float64, device="cuda"),
                         torch.zeros(k, d, dtype=torch.float64, device="cuda")), cfg, np.random.default_rng(3),
                        CudaBackend(k, d, 0.99, 1e-5))
    for _ in range(3):
        vq.step(x, [n])
    xh = x.cpu().pin_memory()
    vq.step(xh, [n])                        # host batch: the H2D pipelined path
    out[name + "_E"] = vq.state[0].cpu().numpy()
    out[name + "_N"] = vq.state[1].cpu().numpy()
np.savez(sys.argv[2], **out)
'''


def _run(env_extra, path):
    env = dict(os.environ)
    env.update(env_extra)
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT, path], env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return np.load(path)


def test_many_chunk_screen_matches_single_chunk(cuda, tmp_path):
    one = _run({}, str(tmp_path / "one.npz"))
    many = _run({"XGS_SCREEN_CHUNK_ROWS": "4096"}, str(tmp_path / "many.npz"))
    for k in one.files:
        assert np.array_equal(one[k], many[k]), k
