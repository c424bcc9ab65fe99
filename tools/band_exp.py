"""Re-rank / fallback row counts over 6 online steps on 2M C5 rows.  The
wider-band emulation in DESIGN.md §10 ran it with a temporary local patch of
capi.cu's screen_args (c1 scaled by XGS_BAND_SCALE); without that patch the
variable has no effect and this prints the true band's counts."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import bench
import paper_2603_09632_b200 as xv
from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
x, E0 = bench.c5_data(torch, 0, 1, dev)
x = x[:1 << 21].contiguous()
cfg = xv.VqConfig(K=bench.C5_K, lam=bench.LAM, gamma=0.5 / bench.C5_K, delta_dead=bench.DELTA, epsilon=bench.EPS, reservoir_capacity=bench.CAP)
be = CudaBackend(bench.C5_K, bench.C5_D, bench.LAM, bench.EPS)
vq = DataParallelVQ((E0, torch.zeros(bench.C5_K, dtype=torch.float64, device=dev), torch.zeros(bench.C5_K, bench.C5_D, dtype=torch.float64, device=dev)), cfg, np.random.default_rng(42), be)
for it in range(6):
    vq.step(x, [int(x.shape[0])])
    cb = xv.Codebook._make(vq.state[0], vq.state[1], vq.state[2], bench.LAM, bench.EPS, None)
    _, (nr, nf) = xv.vq.assign_batch_stats(x, cb)
    print("band", os.environ.get("XGS_BAND_SCALE", "1"), "step", it, "rerank rows", nr, "fallback", nf, flush=True)
