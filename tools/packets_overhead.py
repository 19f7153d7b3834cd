"""Where the per-call time of hamming_decode_packets goes (M, t, P):
events around (a) the whole call, (b) the call captured in a CUDA graph and
replayed, (c) a 16-byte memset alone, (d) K calls back to back / K.
    python tools/packets_overhead.py [M t P]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

M, t = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (400, 5)
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 19
rx, _ = ham.packet_channel_generate(M, t, 3, 0, P, p=1.0)
out = torch.empty(P * M, dtype=torch.uint8, device="cuda")
cnt = torch.empty(2, dtype=torch.int64, device="cuda")


def timed(fn, reps=10):
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts), min(ts)


call = lambda: ham.decode_packets(M, t, rx, P, msg_out=out)  # noqa: E731
call()
torch.cuda.synchronize()
print("call          median/min us: %.1f / %.1f" % timed(call))
print("memset 16 B   median/min us: %.1f / %.1f" % timed(lambda: cnt.zero_()))
K = 8
print("%d calls / %d   median/min us: %.1f / %.1f" % ((K, K) + tuple(x / K for x in timed(lambda: [call() for _ in range(K)]))))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    call()
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    call()
torch.cuda.synchronize()
print("graph replay  median/min us: %.1f / %.1f" % timed(g.replay))
