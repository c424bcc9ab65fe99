"""C4 stream sub-benchmark alone (bench.run_stream)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

import gc

gc.collect()
gc.disable()   # as bench.main: no cyclic-GC pauses inside the timed regions

frames = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
torch.cuda.set_device(0)
print(json.dumps(bench.run_stream(torch, frames, torch.device("cuda", 0))))
