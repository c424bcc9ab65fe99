"""Static instruction count of a kernel's loops (cuobjdump -sass of an object):
python tools/sass_loop.py <obj> <kernel-name-substring>.  Prints each backward
branch (loop) with its body size and an opcode histogram of the largest body."""
import re, subprocess, sys
from collections import Counter

obj, name = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
for f in sass.split("Function : ")[1:]:
    if name not in f.splitlines()[0]:
        continue
    ins = []
    for l in f.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(f.splitlines()[0][:120], len(ins), "instructions")
    loops = []
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s.*?0x([0-9a-f]+)$", t)
        if m and int(m.group(1), 16) < a:
            loops.append((int(m.group(1), 16), a))
    for b, e in loops:
        print(f"  loop {b:#x}..{e:#x}: {(e - b) // 16 + 1} instructions")
    if loops:
        b, e = max(loops, key=lambda x: x[1] - x[0])
        c = Counter()
        for a, t in ins:
            if b <= a <= e:
                op = t.split()[1] if t.startswith("@") else t.split()[0]
                c[op] += 1
        print("  ", ", ".join(f"{k} {v}" for k, v in c.most_common(25)))
