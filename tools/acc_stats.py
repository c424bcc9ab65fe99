"""Per-code row counts of the C2 bench batch after a few steps (how long the
longest accumulate chain is) and the chain kernel time.

    python tools/acc_stats.py [steps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def main():
    import torch
    import paper_2603_09632_b200 as xv
    from paper_2603_09632_b200 import _native as nat
    from paper_2603_09632_b200.distributed import CudaBackend, DataParallelVQ
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    dev = torch.device("cuda", 0)
    x, E0 = bench.make_data(torch, 0, dev)
    cfg = xv.VqConfig(K=bench.K, lam=bench.LAM, gamma=0.5 / bench.K, delta_dead=bench.DELTA, epsilon=bench.EPS,
                      reservoir_capacity=bench.CAP)
    state = (E0.clone(), torch.zeros(bench.K, dtype=torch.float64, device=dev),
             torch.zeros(bench.K, bench.D, dtype=torch.float64, device=dev))
    vq = DataParallelVQ(state, cfg, np.random.default_rng(12), CudaBackend(bench.K, bench.D, bench.LAM, bench.EPS))
    for _ in range(steps):
        vq.step(x, [bench.N_ROWS])
    torch.cuda.synchronize()
    nat.profile_enable(True)
    for _ in range(5):
        vq.step(x, [bench.N_ROWS])
    torch.cuda.synchronize()
    prof = {t: nat.profile_read(t) for t in ("vq_prep", "vq_screen", "vq_accumulate", "vq_chain")}
    nat.profile_enable(False)
    cb = xv.Codebook._make(vq.state[0], vq.state[1], vq.state[2], bench.LAM, bench.EPS, None)
    codes = xv.assign_batch(x, cb)
    c = torch.bincount(codes, minlength=bench.K).cpu().numpy()
    q = np.percentile(c, [0, 50, 90, 99, 100])
    print({"max": int(c.max()), "mean": float(c.mean()), "p0/50/90/99/100": [int(v) for v in q],
           "empty": int((c == 0).sum()), "top8": sorted(c.tolist())[-8:]})
    print({t: (m / max(1, n), n) for t, (m, n) in prof.items()})


if __name__ == "__main__":
    main()
