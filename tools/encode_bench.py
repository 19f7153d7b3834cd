"""Device-timed throughput of the encoder and the SECDED
encoder: min of 8 launches on 2 GiB of coded output per m.
    python tools/encode_bench.py [--m 3 4 5 6] [--gib 2]"""
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
a = ap.parse_args()
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for secded in (False, True):
    for m in a.m:
        n, k = ham.code_nk(m)
        w = (n + 1) if secded else n
        N = int(a.gib * (1 << 30) * 8) // w // 1024 * 1024
        data = torch.randint(0, 256, (ham.data_bytes(m, N),), dtype=torch.uint8, device="cuda")
        enc = ham.encode_secded if secded else ham.encode
        out = enc(m, data, N)
        torch.cuda.synchronize()
        ts = []
        for _ in range(8):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            enc(m, data, N, rx_out=out)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) / 1e3)
        t = min(ts)
        by = ham.data_bytes(m, N) + (ham.secded_coded_bytes(m, N) if secded else ham.coded_bytes(m, N))
        print(f"{'secded ' if secded else ''}encode m={m} N={N} t={t * 1e3:.3f}ms {w * N / t / 1e9:.0f} coded Gbit/s "
              f"{by / t / 1e9:.0f} GB/s ({by / t / 1e9 / peak:.3f})", flush=True)
        del data, out
        torch.cuda.empty_cache()
