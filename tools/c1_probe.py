"""C1 / small-call latency in one process, as bench.py's c1 sweep measures it: a single (7,4) 4 KB
call (queued sleep ahead, median of 100) and 1000 distinct 4 KB packets captured in one CUDA graph
(per packet, best of 5 replays); plus 64 KiB (15,11) calls graph-batched.
python tools/c1_probe.py [tag]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else ""
dev = torch.device("cuda", 0)
st = torch.cuda.current_stream(dev)
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def graph_batched(m, N, G=1000):
    cbp = (ham.coded_bytes(m, N) + 255) // 256 * 256
    dbp = (ham.data_bytes(m, N) + 255) // 256 * 256
    sp = (N + 255) // 256 * 256
    rx = ham.channel_generate(m, 7, 0, N, p=0.1)
    big = torch.empty(G * cbp, dtype=torch.uint8, device=dev)
    big.view(G, cbp)[:, : ham.coded_bytes(m, N)] = rx[: ham.coded_bytes(m, N)]
    bd = torch.empty(G * dbp, dtype=torch.uint8, device=dev)
    bs = torch.empty(G * sp, dtype=torch.uint8, device=dev)
    bc = torch.empty(G, dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(st)
    with torch.cuda.stream(side):
        for i in range(3):
            ham.decode(m, big[i * cbp:], N, data_out=bd[i * dbp:], syndromes=bs[i * sp:], corrected=bc[i:i + 1])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for i in range(G):
                ham.decode(m, big[i * cbp:], N, data_out=bd[i * dbp:], syndromes=bs[i * sp:], corrected=bc[i:i + 1])
    torch.cuda.synchronize()
    g.replay()
    tg = []
    for _ in range(5):
        a, b = ev(), ev()
        a.record(st)
        g.replay()
        b.record(st)
        torch.cuda.synchronize()
        tg.append(a.elapsed_time(b) / 1e3 / G)
    # correctness of the graph-batched outputs: every packet decoded the same input
    ref = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    db = ham.data_bytes(m, N)
    ok = bool((bd.view(G, dbp)[:, :db] == ref.data[:db]).all().item()) and bool((bc == ref.corrected).all().item())
    return min(tg), ok


def single(m, N, reps=100):
    rx = ham.channel_generate(m, 7, 0, N, p=0.1)
    r = ham.decode(m, rx, N)
    ts = []
    for _ in range(reps):
        torch.cuda._sleep(100000)
        a, b = ev(), ev()
        a.record(st)
        ham.decode(m, rx, N, data_out=r.data, syndromes=r.syndromes, corrected=r.corrected)
        b.record(st)
        ts.append((a, b))
    torch.cuda.synchronize()
    xs = sorted(a.elapsed_time(b) for a, b in ts)
    return xs[len(xs) // 2] / 1e3


for m, N, label in ((3, 4681, "C1 (7,4) 4 KB"), (4, 65536 * 8 // 15, "(15,11) 64 KiB"), (4, 546, "(15,11) 1 KiB")):
    t1 = single(m, N)
    tb, ok = graph_batched(m, N)
    print(f"{tag} {label}: single {t1 * 1e6:.2f} us, graph-batched {tb * 1e6:.3f} us per packet, outputs ok={ok}", flush=True)
