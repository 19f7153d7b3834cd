"""Quick device-timed decode throughput (min of 8 launches) for tuning.

    python tools/quick_bench.py [--m 3 4 5 6] [--gib 2] [--reps 8]
Not the benchmark of record (that is bench.py)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, nargs="+", default=[3, 4, 5, 6])
ap.add_argument("--gib", type=float, default=2.0)
ap.add_argument("--reps", type=int, default=8)
ap.add_argument("--tag", default="")
ap.add_argument("--secded", action="store_true", help="extended Hamming (2^m, 2^m-1-m) codewords")
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for m in a.m:
    n, k = ham.code_nk(m)
    if a.secded:
        n = n + 1
    N = int(a.gib * (1 << 30) * 8) // n // 1024 * 1024
    if a.secded:
        rx = ham.channel_generate_secded(m, 1, 0, N, p=0.1, q2=0.1)
        res = ham.decode_secded(m, rx, N)
        res.syndromes, res.corrected = res.flags, res.counts
    elif m <= 6:
        rx = ham.channel_generate(m, 1, 0, N, p=0.1)
        res = ham.decode(m, rx, N)
    else:  # no GPU generator for m = 7, 8: random received bits (decode is branch-free)
        rx = torch.randint(0, 256, (ham.coded_bytes(m, N),), dtype=torch.uint8, device="cuda")
        res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    for syn in (True, False):
        ts = []
        for _ in range(a.reps):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(50000)  # the host's enqueue of the call stays out of the events
            s.record()
            if a.secded:
                ham.decode_secded(m, rx, N, data_out=res.data, flags=res.syndromes if syn else False,
                                  counts=res.corrected)
            else:
                ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes if syn else False,
                           corrected=res.corrected)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        t = min(ts) / 1e3
        by = (ham.secded_coded_bytes(m, N) if a.secded else ham.coded_bytes(m, N)) + ham.data_bytes(m, N) + \
            (N if syn else 0)
        print(f"{a.tag} m={m} syn={syn} N={N} t={t * 1e3:.3f}ms {n * N / t / 1e9:.0f} Gbit/s "
              f"{by / t / 1e9:.0f} GB/s ({by / t / 1e9 / peak:.3f}) grid={ham.last_grid_blocks()}", flush=True)
    del rx, res
    torch.cuda.empty_cache()
