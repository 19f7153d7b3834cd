"""Per-source-line instruction and stall-sample shares from an ncu report
(`ncu -i R --page source --csv --print-source cuda,sass`); usage:
python tools/ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr = None, None
agg, samp, src = collections.Counter(), collections.Counter(), {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    ie, sm = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")

    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    agg[(cur_file, ln)] += num(r[ie])
    samp[(cur_file, ln)] += num(r[sm])
    src[(cur_file, ln)] = r[1][:110]
tot, ts = sum(agg.values()) or 1, sum(samp.values()) or 1
print(f"instructions executed (warp): {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / tot * 100:5.1f}% inst {samp[k] / ts * 100:5.1f}% stall-samples  {k[0]}:{k[1]}  {src[k]}")
