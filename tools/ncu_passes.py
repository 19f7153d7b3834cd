"""Executed warp instructions per pass of packets_decode_kernel, from an ncu
report's source page: python tools/ncu_passes.py report.ncu-rep [n_packets].
Pass boundaries are found by their comment markers in packets.cuh."""
import collections
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = open(os.path.join(ROOT, "paper_1412_6862_b200", "csrc", "packets.cuh")).read().split("\n")
marks = [("S", "group_syndrome64(const uint32_t* w"), ("divmod", "uint32_t divmod_small("),
         ("kernel-setup", "packets_decode_kernel(const"), ("wait", "mbar_wait(&bars[buf]"),
         ("S", "pass S: per (packet, segment) item"), ("X", "if constexpr (HX) {"), ("R", "pass R: every word"),
         ("H", "pass H: head words"),
         ("prefetch", "buffer consumed: prefetch"), ("store", "write the batch's messages"),
         ("tail", "if (lane == 0) bulk_wait<0>();  // the last bulk")]
starts = []
for name, pat in marks:
    ln = next((i + 1 for i, l in enumerate(src) if pat in l), None)
    if ln is not None:
        starts.append((ln, name))
starts.sort()


def which(f, ln):
    if f != "packets.cuh":
        return "other:" + f
    name = "pre"
    for s, n in starts:
        if ln >= s:
            name = n
    return name


out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = collections.Counter()
f = None
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not r[0]:
        continue  # a SASS row (its source line's row carries the totals)
    try:
        ln = int(r[0])
        v = float(r[hdr.index("Instructions Executed")])
    except (ValueError, TypeError):
        continue
    agg[which(f, ln)] += v
P = float(sys.argv[2]) if len(sys.argv) > 2 else 1 << 19
tot = sum(agg.values())
print(f"total {tot:.0f} warp instructions = {tot / P:.1f} per packet")
for k, v in agg.most_common():
    print(f"  {k:16s} {v / tot * 100:5.1f}%  {v / P:7.1f} per packet")
