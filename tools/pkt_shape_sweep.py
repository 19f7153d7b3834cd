"""Forced packet launch shapes in ONE warm process (a -DHAM_PKT_TUNE build reads HAM_PKT_W /
HAM_PKT_G from the environment at every call): python tools/pkt_shape_sweep.py <lib.so> [M t ...]
Prints the fraction of the copy peak per (warps per CTA, packets per batch), plus the model's
own choice ("model") timed in the same process."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["HAMMING_LIB"] = sys.argv[1]
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1412_6862_b200 as ham  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
args = [int(x) for x in sys.argv[2:]] or [400, 5, 400, 2, 800, 6, 1200, 2, 2000, 3]
cells = list(zip(args[0::2], args[1::2]))
P = 1 << 19


def timed(M, t, rx, out, reps=6):
    ham.decode_packets(M, t, rx, P, msg_out=out)
    ts = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(100000)
        s.record()
        ham.decode_packets(M, t, rx, P, msg_out=out)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e) / 1e3)
    return min(ts)


for M, t in cells:
    cb = ham.packet_coded_bytes(M, t)
    rx, _ = ham.packet_channel_generate(M, t, 3, 0, P, p=1.0)
    out = torch.empty(P * M, dtype=torch.uint8, device="cuda")
    alg = P * (cb + M + 2 * t + 1)
    for k in ("HAM_PKT_W", "HAM_PKT_G"):
        os.environ.pop(k, None)
    tm = timed(M, t, rx, out)
    print(f"M={M} t={t} model {ham.packet_launch_shape(M, t, P)}: {alg / tm / 1e9 / PEAK:.3f}", flush=True)
    for w in (4, 8, 12, 16):
        row = []
        for G in (2, 3, 4, 6, 8, 10, 12, 16, 24):
            os.environ["HAM_PKT_W"], os.environ["HAM_PKT_G"] = str(w), str(G)
            try:
                tm = timed(M, t, rx, out)
                row.append(f"G{G}:{alg / tm / 1e9 / PEAK:.3f}/{ham.last_grid_blocks()}")
            except Exception as ex:  # noqa: BLE001
                row.append(f"G{G}:-")
        print(f"  w={w:2d} " + " ".join(row), flush=True)
    del rx, out
    torch.cuda.empty_cache()
