"""C3 grid sub-benchmark alone (bench.run_grid without the CPU leg): prints the per-voxel-size JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

import gc

gc.collect()
gc.disable()   # as bench.main: no cyclic-GC pauses inside the timed regions

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
out = bench.run_grid(torch, steps, cpu=False)
for v, g in out.items():
    if not isinstance(g, dict):
        continue
    print(v, json.dumps({k: g[k] for k in ("Mpts_per_s", "ms_per_batch", "ms_per_batch_python_call",
                                            "ms_per_batch_events", "items_inserted", "batch_voxels", "new_voxels",
                                            "rejected_frac", "map_voxels_before", "map_scene_voxels", "graph",
                                            "map_warm_frames", "per_stage_ms", "batch_hbm_frac")}),
          "front_frac", g["roofline"]["frac"])
