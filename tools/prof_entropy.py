"""Profiling driver: semantic_entropy over 2^21 x 512 fp64 logits (bench consumers workload)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_09632_b200 import thinker as xt

g = torch.Generator(device="cuda")
g.manual_seed(60)
L = torch.randn(1 << 21, 512, generator=g, device="cuda", dtype=torch.float64) * 2.0
for _ in range(2):
    xt.semantic_entropy(L)
torch.cuda.synchronize()
print("done")
