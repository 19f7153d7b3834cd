"""B200 analog of the paper's Table 1 (GPU-over-CPU speedup for
M = 400..2000 bytes x t = 2..6) -- CONTEXT ONLY, not a target.

For each (M, t): a batch of P received packets (one error per segment, the
paper's regime) decoded by hamming_decode_packets (device-timed, inputs in
HBM), against the CPU oracle decoding the same packets on ONE host thread
(the paper's "equivalent sequential approach") and on all host
threads.  Prints a markdown table."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: timed baseline only)
import paper_1412_6862_b200 as ham  # noqa: E402

THREADS = len(os.sched_getaffinity(0))
P_GPU = int(os.environ.get("P_GPU", 1 << 19))
P_CPU = int(os.environ.get("P_CPU", 2000))

rows = []
for M in (400, 800, 1200, 1600, 2000):
    for t in (2, 3, 4, 5, 6):
        stride = ham.packet_stride(M, t)
        cb = ham.packet_coded_bytes(M, t)
        rx, msg = ham.packet_channel_generate(M, t, 0x7AB1E, 0, P_GPU, p=1.0)
        out = torch.empty(P_GPU * M, dtype=torch.uint8, device="cuda")
        ham.decode_packets(M, t, rx, P_GPU, msg_out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            ham.decode_packets(M, t, rx, P_GPU, msg_out=out)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e) / 1e3)
        tg = min(ts) / P_GPU                       # seconds per packet on the GPU (batched)
        alg = cb + M + 2 * t + 1
        # oracle: the same packets (the oracle's own generator), 1 thread and all threads
        rx_c, _ = oracle.generate_packets(M, t, 0x7AB1E, 0, P_CPU, stride, p=1.0, threads=THREADS)
        t0 = time.perf_counter()
        oracle.decode_packets(M, t, rx_c, P_CPU, stride, threads=1)
        t1 = (time.perf_counter() - t0) / P_CPU
        t0 = time.perf_counter()
        oracle.decode_packets(M, t, rx_c, P_CPU, stride, threads=THREADS)
        tT = (time.perf_counter() - t0) / P_CPU
        rows.append((M, t, cb, tg, alg / tg / 1e9, 8 * cb / tg / 1e9, t1, tT))
        print(f"M={M} t={t}: GPU {tg * 1e9:.1f} ns/packet ({alg / tg / 1e9:.0f} GB/s, {8 * cb / tg / 1e9:.0f} coded Gbit/s); "
              f"oracle 1 thread {t1 * 1e6:.1f} us, {THREADS} threads {tT * 1e6:.2f} us; "
              f"speedup {t1 / tg:.0f}x / {tT / tg:.0f}x", flush=True)
        del rx, out
        torch.cuda.empty_cache()

print(f"\n| M (bytes) | t | coded B/packet | GPU ns/packet | GPU GB/s | oracle 1-thread us/packet | speedup vs 1 thread | speedup vs {THREADS} threads |")
print("|---|---|---|---|---|---|---|---|")
for M, t, cb, tg, gbs, gbit, t1, tT in rows:
    print(f"| {M} | {t} | {cb} | {tg * 1e9:.1f} | {gbs:.0f} | {t1 * 1e6:.1f} | {t1 / tg:.0f}x | {tT / tg:.0f}x |")
