"""C1 / C2 (BASELINE.json configs[0], configs[1]): small packets are launch- and
latency-bound, so report (i) single-call device latency (CUDA events around one
hamming_decode, median of 200, L2-warm) and (ii) the throughput of 1000 calls
captured in one CUDA graph on 1000 distinct packets (graph replay time / 1000).
C2 also sweeps the size up to 64 MiB (cold L2 above ~4x L2 is the steady state)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402


def single_latency(m, rx, N, data, syn, cnt, reps=200):
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        ham.decode(m, rx, N, data_out=data, syndromes=syn, corrected=cnt)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) * 1e3)
    return statistics.median(ts)


def graph_batch(m, N, G=1000):
    cb, db = ham.coded_bytes(m, N), ham.data_bytes(m, N)
    cbp, dbp = (cb + 255) // 256 * 256, (db + 255) // 256 * 256
    rx = ham.channel_generate(m, 11, 0, N * 0 + N, p=0.1)
    big_rx = torch.empty(G * cbp, dtype=torch.uint8, device="cuda")
    for i in range(G):
        big_rx[i * cbp: i * cbp + cb] = rx[:cb]
    data = torch.empty(G * dbp, dtype=torch.uint8, device="cuda")
    syn = torch.empty(G * ((N + 255) // 256 * 256), dtype=torch.uint8, device="cuda")
    cnt = torch.empty(G, dtype=torch.int64, device="cuda")
    sp = (N + 255) // 256 * 256
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            ham.decode(m, big_rx[i * cbp:], N, data_out=data[i * dbp:], syndromes=syn[i * sp:], corrected=cnt[i:i + 1])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(G):
                ham.decode(m, big_rx[i * cbp:], N, data_out=data[i * dbp:], syndromes=syn[i * sp:],
                           corrected=cnt[i:i + 1])
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / G)
    return min(ts)


rows = []
# C1: (7,4), one 4 KB packet
m, N = 3, 4681
rx = ham.channel_generate(m, 0x14126862, 0, N, p=0.1)
res = ham.decode(m, rx, N)
lat = single_latency(m, rx, N, res.data, res.syndromes, res.corrected)
gb = graph_batch(m, N)
print(f"C1 (7,4) 4 KB: single-call {lat:.2f} us; CUDA-graph batched {gb:.2f} us/packet "
      f"= {7 * N / gb / 1e3:.1f} coded Gbit/s", flush=True)
rows.append(("C1", 3, 4096, N, lat, gb))
# C2: (15,11) sweep
m = 4
for S in [400, 800, 1200, 1600, 2000] + [1 << e for e in range(10, 27, 2)]:
    N = S * 8 // 15
    rx = ham.channel_generate(m, S, 0, N, p=0.1)
    res = ham.decode(m, rx, N)
    lat = single_latency(m, rx, N, res.data, res.syndromes, res.corrected, reps=100 if S < (1 << 24) else 20)
    gb = graph_batch(m, N, G=200) if S <= (1 << 20) else float("nan")
    alg = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
    print(f"C2 (15,11) {S} B (N={N}): single-call {lat:.2f} us ({15 * N / lat / 1e3:.1f} coded Gbit/s, "
          f"{alg / lat / 1e3:.0f} GB/s); graph-batched {gb:.2f} us", flush=True)
    rows.append(("C2", 4, S, N, lat, gb))
print("\n| config | code | packet bytes (coded) | N | single-call us | coded Gbit/s (single) | graph-batched us/packet | coded Gbit/s (batched) |")
print("|---|---|---|---|---|---|---|---|")
for c, m, S, N, lat, gb in rows:
    n = 2 ** m - 1
    gbs = f"{n * N / gb / 1e3:.1f}" if gb == gb else "-"
    gbt = f"{gb:.2f}" if gb == gb else "-"
    print(f"| {c} | ({n},{n - m}) | {S} | {N} | {lat:.2f} | {n * N / lat / 1e3:.1f} | {gbt} | {gbs} |")
