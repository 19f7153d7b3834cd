"""Top source lines of an ncu report by executed instructions and stall samples:
python tools/ncu_lines_top.py report.ncu-rep [file-substring] [n] [per-unit]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
fsub = sys.argv[2] if len(sys.argv) > 2 else "packets.cuh"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
per = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
f = None
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if f is None or fsub not in f:
        continue
    try:
        ln = int(r[0])
        ins = float(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, TypeError):
        continue
    samp = 0.0
    if not r[0]:
        continue  # a SASS row
    for key in ("Warp Stall Sampling (All Samples)", "Sampling Data (All)"):
        if key in hdr:
            try:
                samp = float(r[hdr.index(key)] or 0)
            except ValueError:
                pass
    rows.append((ins, samp, ln, r[1][:110]))
tot_i = sum(x[0] for x in rows) or 1
tot_s = sum(x[1] for x in rows) or 1
print(f"{fsub}: {tot_i:.0f} instructions, {tot_s:.0f} samples")
for ins, samp, ln, src in sorted(rows, reverse=True)[:N]:
    print(f"{ln:5d} {ins / per:9.1f} {100 * ins / tot_i:5.1f}% samp {100 * samp / tot_s:5.1f}%  {src}")
