"""C3 per-call cost (256 MiB per call) measured several ways, to separate the
kernel from launch gaps, buffer placement and timing artefacts:
  eager-1set   back-to-back calls on one buffer set, events around each call
  eager-2sets  the same alternating between two buffer sets (bench sweeps)
  loop         one event pair around 20 calls (no per-call events)
  graph        20 calls captured in one CUDA graph, replay timed
python tools/c3_probe.py [m ...]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

PEAK = 6544.0
ms = [int(a) for a in sys.argv[1:]] or [3, 4, 5, 6]
st = torch.cuda.current_stream()


def ev():
    return torch.cuda.Event(enable_timing=True)


for m in ms:
    n, k = ham.code_nk(m)
    N = (256 << 20) * 8 // n
    sets = []
    for b in range(2):
        rx = ham.channel_generate(m, 7 + b, 0, N, p=0.1)
        sets.append((rx, torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, device="cuda"),
                     torch.empty(N, dtype=torch.uint8, device="cuda"), torch.empty(1, dtype=torch.int64, device="cuda")))
    for syn_on in (True, False):
        alg = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + (N if syn_on else 0) + 8

        def call(i):
            rx, d, sy, c = sets[i]
            ham.decode(m, rx, N, data_out=d, syndromes=sy if syn_on else False, corrected=c)

        res = {}
        for name, pick in (("eager-1set", lambda i: 0), ("eager-2sets", lambda i: i & 1)):
            for i in range(4):
                call(pick(i))
            evs = []
            for i in range(24):
                a, b = ev(), ev()
                a.record(st)
                call(pick(i))
                b.record(st)
                evs.append((a, b))
            torch.cuda.synchronize()
            ts = [a.elapsed_time(b) * 1e3 for a, b in evs[4:]]
            res[name] = (statistics.median(ts), min(ts))
        a, b = ev(), ev()
        a.record(st)
        for i in range(20):
            call(0)
        b.record(st)
        torch.cuda.synchronize()
        res["loop"] = (a.elapsed_time(b) * 1e3 / 20,) * 2
        s = torch.cuda.Stream()
        s.wait_stream(st)
        with torch.cuda.stream(s):
            call(0)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(20):
                    call(0)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        res["graph"] = (a.elapsed_time(b) * 1e3 / 20,) * 2
        line = " ".join(f"{k}: {v[0]:.1f} us ({alg / v[0] / 1e3 / PEAK:.3f}) min {v[1]:.1f}" for k, v in res.items())
        print(f"m={m} syn={'on ' if syn_on else 'off'} {line}", flush=True)
    del sets
    torch.cuda.empty_cache()
