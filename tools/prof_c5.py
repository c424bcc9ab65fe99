"""Profiling driver: C5-shard online steps (for ncu runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
print(bench.run_c5(torch, int(sys.argv[1]) if len(sys.argv) > 1 else 1, torch.device("cuda", 0))["ms_per_iter"])
