"""Profiling driver: the C4 stream (bench.run_stream) for ncu launch lists."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 40
torch.cuda.set_device(0)
print(json.dumps(bench.run_stream(torch, frames, torch.device("cuda", 0)))[:400])
