"""Tabulate a `tune_shapes.py run packets` log: fraction of the copy peak per (M, t) x variant.
python tools/tune_table.py gpurun_out/tune_pkt13.txt"""
import collections
import re
import sys

cur = None
res = collections.defaultdict(dict)
for line in open(sys.argv[1]):
    if line.startswith("budget"):
        p = line.split()
        cur = f"b{p[1]}w{p[7]}"
    m = re.match(r"M=(\d+) t=(\d+).*\((0\.\d+)\).*grid=(\d+)", line)
    if m:
        res[(int(m[1]), int(m[2]))][cur] = (float(m[3]), int(m[4]))
cols = sorted({c for v in res.values() for c in v}, key=lambda c: (int(c[1:].split("w")[0]), int(c.split("w")[1])))
print("M,t       " + " ".join(f"{c:>12s}" for c in cols) + "   best")
for k in sorted(res):
    row = res[k]
    best = max(row, key=lambda c: row[c][0])
    print(f"{str(k):9s} " + " ".join(f"{row.get(c, (0, 0))[0]:7.3f}/{row.get(c, (0, 0))[1]:<4d}" for c in cols) + f"   {best}")
