"""Which earlier sub-benchmark slows bench.run_raster down in the full bench run?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)


def rr(tag):
    r = bench.run_raster(torch, 3, cpu=False)
    print(tag, round(r["build_ms"], 3), round(r["vjp_ms"], 3), flush=True)


rr("alone")
bench.cpu_port_c5(5.0)
rr("after cpu_port_c5")
bench.run_c1(torch, cpu=False)
rr("after c1")
bench.run_stream(torch, 100, dev)
rr("after stream")
bench.run_grid(torch, 2, cpu=False)
rr("after grid")
