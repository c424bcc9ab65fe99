"""C5 at N=1: all 67,108,864 bf16 rows x 1152, K=4096 on one GPU (bounded screening workspace)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

import gc

gc.collect()
gc.disable()   # as bench.main: no cyclic-GC pauses inside the timed regions

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
torch.cuda.set_device(0)
print(json.dumps(bench.run_c5(torch, iters, torch.device("cuda", 0))), flush=True)
