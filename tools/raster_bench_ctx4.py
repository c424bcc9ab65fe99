"""How long does the host stay slow after the CPU port (bench.cpu_port_c5)?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)


def rr(tag):
    r = bench.run_raster(torch, 3, cpu=False)
    print(tag, round(r["build_ms"], 3), flush=True)


import gc
rr("alone")
for wait in (0, 1, 3, 10):
    if wait == 3:
        gc.collect()
        gc.disable()
        print("gc disabled from here")
    bench.cpu_port_c5(3.0)
    time.sleep(wait)
    rr(f"after cpu_port_c5 + {wait}s")
import threading
print("threads alive", threading.active_count())
