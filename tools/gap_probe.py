"""Per-call cost of back-to-back 256 MiB decodes: eager stream vs one CUDA graph
of the same calls (host enqueue removed).  python tools/gap_probe.py [m] [MiB]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mib = float(sys.argv[2]) if len(sys.argv) > 2 else 256
n, k = ham.code_nk(m)
N = int(mib * (1 << 20) * 8) // n
rx = ham.channel_generate(m, 1, 0, N, p=0.1)
res = ham.decode(m, rx, N)
K = 20


def calls():
    for _ in range(K):
        ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected)


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    calls()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    calls()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"eager: {e0.elapsed_time(e1) * 1e3 / K:.1f} us per call", flush=True)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        calls()
    g.replay()
    torch.cuda.synchronize()
    e0.record(s)
    g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"graph: {e0.elapsed_time(e1) * 1e3 / K:.1f} us per call", flush=True)

# the same on the legacy default stream, and with two events per call (bench.py's pattern)
d = torch.cuda.current_stream()
torch.cuda.synchronize()
e0.record(d)
calls()
e1.record(d)
torch.cuda.synchronize()
print(f"eager, default stream: {e0.elapsed_time(e1) * 1e3 / K:.1f} us per call", flush=True)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
for st, name in ((d, "default"), (s, "side")):
    with torch.cuda.stream(st):
        torch.cuda.synchronize()
        e0.record(st)
        for a, b in evs:
            a.record(st)
            ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected)
            b.record(st)
        e1.record(st)
        torch.cuda.synchronize()
        print(f"eager + events, {name} stream: {e0.elapsed_time(e1) * 1e3 / K:.1f} us per call, "
              f"per-call events {sum(a.elapsed_time(b) for a, b in evs) * 1e3 / K:.1f} us", flush=True)
