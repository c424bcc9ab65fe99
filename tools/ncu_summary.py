"""Summarise ncu captures into profiles/*.md (run here, no GPU needed).

    python tools/ncu_summary.py launches.csv [full.ncu-rep ...] > profiles/rN_ncu_summary.md
"""
import csv
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "time (us)", None),
    ("dram__bytes_read.sum", "DRAM read (MB)", None),
    ("dram__bytes_write.sum", "DRAM write (MB)", None),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak", None),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe (realtime) %", None),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %", None),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %", None),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", None),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %", None),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", None),
    ("launch__registers_per_thread", "regs", None),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    unit = h.index("Metric Unit") if "Metric Unit" in h else None
    per = defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            u = r[unit] if unit is not None else ""
            if u in ("Kbyte", "KB"):
                v *= 1e3
            elif u in ("Mbyte", "MB"):
                v *= 1e6
            elif u in ("Gbyte", "GB"):
                v *= 1e9
            elif u in ("usecond", "us"):
                v *= 1e3
            elif u in ("msecond", "ms"):
                v *= 1e6
            per[(r[ii], r[ki])][r[mi]] = v
    agg = defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in per.items():
        name = k.split("(")[0].replace("xgs::<unnamed>::", "").replace("void ", "")[:60]
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"### Launch list `{path}` (cold-cache, serialised; compare shares)\n")
    print("| kernel | launches | total us | share | DRAM MB | GB/s |")
    print("|---|---|---|---|---|---|")
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {c} | {t/1e3:.1f} | {100*t/tot:.1f}% | {b/1e6:.1f} | {b/t if t else 0:.0f} |")
    print()


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    scale_of = {"ms": 1e3, "msecond": 1e3, "us": 1.0, "usecond": 1.0, "ns": 1e-3, "nsecond": 1e-3,
                "GB": 1e3, "Gbyte": 1e3, "MB": 1.0, "Mbyte": 1.0, "KB": 1e-3, "Kbyte": 1e-3, "byte": 1e-6}

    def col(m):
        for i, n in enumerate(h):
            if n == m or n.endswith("." + m):
                return i
        return None
    print(f"### `ncu --set full` capture `{path}`\n")
    print("| kernel | " + " | ".join(m[1] for m in METRICS) + " |")
    print("|---|" + "---|" * len(METRICS))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("xgs::<unnamed>::", "").replace("void ", "")[:50]
        vals = []
        for m, _, _ in METRICS:
            i = col(m)
            try:
                v = float(r[i].replace(",", "")) * scale_of.get(units[i], 1.0)
                vals.append(f"{v:.1f}")
            except (ValueError, IndexError, TypeError):
                vals.append("-")
        print(f"| `{name}` | " + " | ".join(vals) + " |")
    print()


if __name__ == "__main__":
    for a in sys.argv[1:]:
        (full if a.endswith(".ncu-rep") else launches)(a)
