"""One C2 online_step out of an ncu launch list (gpu__time_duration.sum +
dram bytes per launch): the kernels between two consecutive C2 row-prep
launches, with each kernel's share of the step (cold-cache, serialised
replay: compare shares, not absolute times).

    python tools/launch_step.py gpurun_out/r_launches.csv [which=2]
    python tools/launch_step.py profiles/r1_launches_session3.csv   (slimmed copy)
"""
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    if rows and rows[0][:2] == ["ID", "kernel"]:   # profiles/ copy: one row per launch
        out = []
        for r in rows[1:]:
            m = {"gpu__time_duration.sum": float(r[4] or 0), "dram__bytes_read.sum": float(r[5] or 0),
                 "dram__bytes_write.sum": float(r[6] or 0)}
            out.append([r[1], m])
        return out
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ik, im, iv, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    seq = {}
    for r in rows[hi + 1:]:
        if len(r) != len(h):
            continue
        nm = r[ik].split("(")[0].replace("void ", "").replace("xgs::<unnamed>::", "")
        seq.setdefault(int(r[ii]), [nm, {}])[1][r[im]] = float(r[iv].replace(",", ""))
    return [v for _, v in sorted(seq.items())]


def main():
    seq = load(sys.argv[1])
    which = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    # C2 steps: a >100 us fp32 row prep starts each step's device work
    starts = [i for i, (nm, m) in enumerate(seq)
              if nm.startswith("prep_rows_kernel<float>") and m.get("gpu__time_duration.sum", 0) > 1e5]
    a, b = starts[which], starts[which + 1]
    # include the small codebook-prep kernels that precede the row prep
    while a > 0 and seq[a - 1][0].startswith(("absmax_kernel", "prep_codebook_kernel")):
        a -= 1
    while b > 0 and seq[b - 1][0].startswith(("absmax_kernel", "prep_codebook_kernel")):
        b -= 1
    step = seq[a:b]
    tot = sum(m.get("gpu__time_duration.sum", 0) for _, m in step)
    print("| kernel | us | share | DRAM read MB | DRAM write MB |")
    print("|---|---|---|---|---|")
    for nm, m in step:
        t = m.get("gpu__time_duration.sum", 0)
        print(f"| `{nm[:48]}` | {t / 1e3:.1f} | {100 * t / tot:.1f}% | {m.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
              f"{m.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    print(f"| **sum** | {tot / 1e3:.1f} | 100% | | |")


if __name__ == "__main__":
    main()
