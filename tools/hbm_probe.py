"""HBM reference: torch copy_ throughput, short bursts vs sustained, and the
decode kernel's per-step times over a long back-to-back run (is the sustained
rate a power/thermal effect or the memory system's steady state?)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return ts


for gib in (1, 32):
    n = gib << 30
    a = torch.empty(n, dtype=torch.uint8, device="cuda")
    b = torch.empty(n, dtype=torch.uint8, device="cuda")
    a.fill_(1)
    reps = 10 if gib == 1 else 40
    ts = timed(lambda: b.copy_(a), reps)
    bw = [2 * n / (t / 1e3) / 1e9 for t in ts]
    print(f"copy {gib} GiB x{reps}: best {max(bw):.0f} GB/s, first {bw[0]:.0f}, last {bw[-1]:.0f}, "
          f"mean {sum(bw) / len(bw):.0f} GB/s", flush=True)
    del a, b
    torch.cuda.empty_cache()

m = 6
N = (1 << 39) // 63
rx = ham.channel_generate(m, 1, 0, N, p=0.1)
res = ham.decode(m, rx, N)
torch.cuda.synchronize()
alg = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
ts = timed(lambda: ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected), 40)
bw = [alg / (t / 1e3) / 1e9 for t in ts]
print("decode C5 per-step GB/s:", " ".join(f"{x:.0f}" for x in bw), flush=True)
time.sleep(2)
ts = timed(lambda: ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected), 5)
print("after 2 s idle:", " ".join(f"{alg / (t / 1e3) / 1e9:.0f}" for t in ts), flush=True)
