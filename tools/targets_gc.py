"""bench.run_targets repeated after run_stream (is the slowdown persistent or transient?)."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
gc.disable()
for i in range(3):
    print("alone", round(bench.run_targets(torch, 10, cpu=False)["ms_per_keyframe"], 3))
bench.run_stream(torch, 100, dev)
gc.collect()
for i in range(5):
    print("after stream", i, round(bench.run_targets(torch, 10, cpu=False)["ms_per_keyframe"], 3))
torch.cuda.empty_cache()
for i in range(3):
    print("after empty_cache", i, round(bench.run_targets(torch, 10, cpu=False)["ms_per_keyframe"], 3))
time.sleep(5)
print("after 5 s idle", round(bench.run_targets(torch, 10, cpu=False)["ms_per_keyframe"], 3))
