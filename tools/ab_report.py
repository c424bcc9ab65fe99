"""Summarise tools/gpu_ab.sh output: per variant and pass, sync / graph ms and the front-end stage."""
import glob, json, os, re
for f in sorted(glob.glob("gpurun_out/ab_tests_*.log")):
    print(os.path.basename(f), open(f).read().strip().splitlines()[-1])
for f in sorted(glob.glob("gpurun_out/ab_*_[0-9].log")):
    for l in open(f):
        if l[:4] in ("0.01", "0.05"):
            v, rest = l.split(" ", 1)
            d = json.loads(rest[:rest.rindex("}") + 1])
            print(os.path.basename(f)[3:-4], v, round(d["ms_per_batch"], 4), round(d["graph"]["ms_per_batch"], 4),
                  round(d["per_stage_ms"]["grid_keys"], 4))
for f in sorted(glob.glob("gpurun_out/abs_*_[0-9].log")):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(os.path.basename(f)[4:-4], "C4 p50", round(d["p50_ms"], 4), "p99", round(d["p99_ms"], 4),
                  "mean", round(d["mean_ms"], 4))
