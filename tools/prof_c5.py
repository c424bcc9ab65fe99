"""Profiling driver: C5 per-GPU shard online_steps (for ncu runs).

    python tools/prof_c5.py [iters=1]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 1
torch.cuda.set_device(0)
print(bench.run_c5(torch, iters, torch.device("cuda", 0)))
