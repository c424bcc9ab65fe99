"""Timeline of the row-chunk pipelined VQ step at C2 (profiling aid).

    XGS_PIPE_CHUNKS=8 python tools/pipe_timeline.py out.csv
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2603_09632_b200 import _native as nat
from paper_2603_09632_b200 import vq as xvq

torch.cuda.set_device(0)
x, E0 = bench.make_data(torch, 0, torch.device("cuda", 0))
K, D = bench.K, bench.D
r, dt, n, d, ldx = xvq._rows(x)
for _ in range(3):
    xvq._assign_accumulate_dev(r, dt, n, d, ldx, E0, K)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for _ in range(5):
    xvq._assign_accumulate_dev(r, dt, n, d, ldx, E0, K)
ev[1].record()
torch.cuda.synchronize()
print("chunks", os.environ.get("XGS_PIPE_CHUNKS", "auto"), "ms/step", ev[0].elapsed_time(ev[1]) / 5)
nat.lib().xgs_profile_enable(1)
xvq._assign_accumulate_dev(r, dt, n, d, ldx, E0, K)
torch.cuda.synchronize()
nat.lib().xgs_profile_dump(sys.argv[1].encode())
