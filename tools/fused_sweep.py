"""Forced launch shapes of the fused packet decoder in ONE warm process (a -DHAM_PKT_TUNE build
reads HAM_FUSED_L / HAM_FUSED_G / HAM_FUSED_W at every call; HAM_PKT_SPLIT=1 selects the split
multi-pass decoder): python tools/fused_sweep.py <lib.so> [M t ...].  Prints, per (M, t), the
fraction of the copy peak of the model's shape, of the split decoder, and of each forced shape."""
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
KEYS = ("HAM_FUSED_L", "HAM_FUSED_G", "HAM_FUSED_W", "HAM_FUSED_S", "HAM_PKT_SPLIT")


def timed(M, t, rx, out, reps=5):
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
    for k in KEYS:
        os.environ.pop(k, None)
    frac = lambda tm: alg / tm / 1e9 / PEAK  # noqa: E731
    model = ham.packet_launch_shape(M, t, P)
    fm = frac(timed(M, t, rx, out))
    os.environ["HAM_PKT_SPLIT"] = "1"
    fs = frac(timed(M, t, rx, out))
    os.environ.pop("HAM_PKT_SPLIT")
    print(f"M={M} t={t} model L={model['lanes_per_item']} G={model['packets_per_batch']} "
          f"w={model['warps']}x{model['ctas_per_sm']}: fused {fm:.3f}  split {fs:.3f}", flush=True)
    best = (0, None)
    for L in (1, 2, 4, 8):
        for S in (2, 3, 4):
            for w in (4, 8):
                row = []
                for G in (2, 3, 4, 6, 8, 12, 16):
                    os.environ.update(HAM_FUSED_L=str(L), HAM_FUSED_W=str(w), HAM_FUSED_G=str(G), HAM_FUSED_S=str(S))
                    try:
                        f = frac(timed(M, t, rx, out, reps=3))
                        row.append(f"{G}:{f:.3f}")
                        if f > best[0]:
                            best = (f, (L, S, w, G))
                    except Exception:  # noqa: BLE001 -- shape does not fit / not legal
                        row.append(f"{G}:--")
                print(f"  L={L} S={S} w={w}: " + " ".join(row), flush=True)
    for k in KEYS:
        os.environ.pop(k, None)
    print(f"  best {best[0]:.3f} at L,S,w,G={best[1]}", flush=True)
    del rx, out
    torch.cuda.empty_cache()
