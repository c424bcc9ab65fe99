"""C4: host cost of the per-frame graph launch -- torch's CUDAGraph.replay() against
cudaGraphLaunch on its raw exec handle (ctypes, the runtime torch loads); p50 of the
stream bench either way.  Profiling aid."""
import ctypes
import glob
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
import paper_2603_09632_b200.stream as S

import gc

gc.collect()
gc.disable()
mode = sys.argv[1] if len(sys.argv) > 1 else "torch"
import nvidia
rt = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(nvidia.__path__[0]), "nvidia", "cuda_runtime", "lib",
                                        "libcudart.so.12"))[0])
rt.cudaGraphLaunch.argtypes = [ctypes.c_void_p, ctypes.c_void_p]


class Direct:
    def __init__(self, g):
        self.g, self.exec = g, ctypes.c_void_p(g.raw_cuda_graph_exec())

    def replay(self):
        rc = rt.cudaGraphLaunch(self.exec, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        if rc:
            raise RuntimeError(f"cudaGraphLaunch {rc}")


if mode == "direct":
    _cap = S.PerceiverStream._capture

    def cap(self):
        _cap(self)
        self.graphs = [Direct(g) for g in self.graphs]
        self.graph = self.graphs[0]
    S.PerceiverStream._capture = cap
torch.cuda.set_device(0)
r = bench.run_stream(torch, 1000, torch.device("cuda", 0))
print(mode, json.dumps({k: r[k] for k in ("p50_ms", "p99_ms", "mean_ms", "graph_frames")}))
