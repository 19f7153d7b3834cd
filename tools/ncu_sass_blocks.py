"""Basic blocks of the profiled kernel's SASS ranked by executed warp
instructions (ncu source page, sass view): python tools/ncu_sass_blocks.py R [top] [lines]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
show = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
data = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
ie, src, smp = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")


def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


tot = sum(num(r[ie]) for r in data) or 1
segs, cur, start, acc = [], None, 0, 0
for i, r in enumerate(data):
    c = num(r[ie])
    if c != cur:
        if cur is not None:
            segs.append((acc, cur, start, i - 1))
        cur, start, acc = c, i, 0
    acc += c
segs.append((acc, cur, start, len(data) - 1))
print(f"total warp instructions {tot}")
for acc, c, a, b in sorted(segs, reverse=True)[:top]:
    print(f"{acc / tot * 100:5.1f}%  x{c}  [{a}..{b}] {b - a + 1} instr")
    for r in data[a:min(b + 1, a + show)]:
        print("      ", r[src].strip()[:90], r[smp])
