"""What a plain device copy of the same bytes reaches at C3's per-call size.

For each m, a D2D copy moving the same algorithmic bytes as one 256 MiB decode
call (read coded_bytes, write data_bytes + N syndrome bytes), timed like
bench.py's C3 sweep (median of 20 back-to-back calls alternating between two
buffer sets, CUDA events on the current stream).  The copy is torch's
(cudaMemcpyAsync D2D), i.e. the same primitive MEASURED_PEAKS uses at 2 GiB --
the per-call ceiling a single-kernel decode of this size can hope for.
    python tools/copy_ceiling.py [--mib 256]
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mib", type=float, nargs="+", default=[256.0])
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
for mib in a.mib:
    for m in (3, 4, 5, 6):
        n, k = ham.code_nk(m)
        N = int(mib * (1 << 20) * 8) // n
        rd = ham.coded_bytes(m, N)
        wr = ham.data_bytes(m, N) + N
        # a copy reads and writes the same count: copy max(rd, wr)/... -> copy (rd+wr)/2 bytes
        half = (rd + wr) // 2 // 16 * 16
        bufs = [(torch.empty(half, dtype=torch.uint8, device="cuda"), torch.empty(half, dtype=torch.uint8, device="cuda"))
                for _ in range(2)]
        for s, d in bufs:
            d.copy_(s)
        torch.cuda.synchronize()
        ts = []
        for i in range(a.reps):
            s, d = bufs[i & 1]
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            d.copy_(s)
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        us = statistics.median(e0.elapsed_time(e1) * 1e3 for e0, e1 in ts)
        gbs = 2 * half / us / 1e3
        print(json.dumps({"mib": mib, "m": m, "bytes_per_call": 2 * half, "us_per_call": round(us, 2),
                          "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}), flush=True)
        del bufs
        torch.cuda.empty_cache()
