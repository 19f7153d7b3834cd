"""Device-timed throughput of hamming_decode_packets for one (M, t).

Each timed call is preceded by a queued sleep kernel (torch.cuda._sleep), so
the host's enqueue time of the call (the Python binding + the C ABI's launch)
is not inside the events: an idle stream would otherwise start the first
event the moment it is recorded and count ~20 us of host work as device time
(tools/packets_overhead.py: single call 126.6 us vs 102.7 us back to back for
M = 400, t = 5, 2^19 packets)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, nargs="+", default=[2000])
ap.add_argument("--t", type=int, nargs="+", default=[2])
ap.add_argument("--P", type=int, default=1 << 19)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for M in a.M:
    for t in a.t:
        cb = ham.packet_coded_bytes(M, t)
        rx, _ = ham.packet_channel_generate(M, t, 3, 0, a.P, p=1.0)
        out = torch.empty(a.P * M, dtype=torch.uint8, device="cuda")
        ham.decode_packets(M, t, rx, a.P, msg_out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(a.reps):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(50000)  # keeps the stream busy while the host enqueues the call
            s.record()
            ham.decode_packets(M, t, rx, a.P, msg_out=out)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) / 1e3)
        tm = min(ts)
        alg = a.P * (cb + M + 2 * t + 1)
        print(f"M={M} t={t} P={a.P}: {tm * 1e3:.3f} ms, {alg / tm / 1e9:.0f} GB/s ({alg / tm / 1e9 / PEAK:.3f}), "
              f"{8 * cb * a.P / tm / 1e9:.0f} coded Gbit/s, grid={ham.last_grid_blocks()}", flush=True)
        del rx, out
        torch.cuda.empty_cache()
