"""Profiling driver: relevance_per_gaussian at the C4 map size (2^21 x K=512, D=768) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_09632_b200 import core
import paper_2603_09632_b200.thinker as xt

n, K, D = 1 << 21, 512, 768
g = torch.Generator(device="cuda")
g.manual_seed(0)
L = 2.0 * torch.randn(n, K, generator=g, device="cuda", dtype=torch.float64)
E = torch.randn(K, D, generator=g, device="cuda", dtype=torch.float64)
Q = torch.randn(5, D, generator=g, device="cuda", dtype=torch.float64)
Q /= Q.norm(dim=1, keepdim=True)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    core.gemm_f64(L, E, softmax=True, query=Q, tau=10.0, eps=1e-8, want_c=False)
torch.cuda.synchronize()
print("done")
