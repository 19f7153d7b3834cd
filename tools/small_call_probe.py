"""Where a single small decode call's ~10 us goes: events around 1, 2 and 8 back-to-back calls
of a (15,11) 400-byte packet after a long queued sleep, an empty torch kernel for comparison,
and (under ncu) the kernel's own duration.   python tools/small_call_probe.py"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

m, N = 4, 213
rx = ham.channel_generate(m, 5, 0, N, p=0.1)
d = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, device="cuda")
sy = torch.empty(N, dtype=torch.uint8, device="cuda")
c = torch.empty(1, dtype=torch.int64, device="cuda")
x = torch.empty(16, device="cuda")


def run(k, fn, reps=30):
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(300000)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts)


dec = lambda: ham.decode(m, rx, N, data_out=d, syndromes=sy, corrected=c)  # noqa: E731
dec()
torch.cuda.synchronize()
for k in (1, 2, 8):
    print(f"decode x{k}: {run(k, dec):.2f} us  ({run(k, dec) / k:.2f} per call)")
print(f"torch x.add_(1) x1: {run(1, lambda: x.add_(1)):.2f} us, x8: {run(8, lambda: x.add_(1)) / 8:.2f} per call")
print(f"nothing: {run(1, lambda: None):.2f} us")
