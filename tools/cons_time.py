"""Consumers sub-benchmark repeated in one process (first-call effects)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    r = bench.run_consumers(torch, 5, cpu=False)
    print(json.dumps({"entropy_ms": r["semantic_entropy"]["ms"], "tokens_ms": r["sample_tokens"]["ms"],
                      "relevance_ms": r["relevance_per_gaussian"]["ms"], "sm_mhz": r["clocks"]["sm_mhz"]}))
