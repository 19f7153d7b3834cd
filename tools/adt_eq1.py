"""The paper's transfer model (Eq. 1) checked on
the B200 host link with the library's own pipeline, hamming_decode_host:

  T_PS   H2D copy of one chunk's packet bytes (pinned host -> device)
  T_DKE  the decode kernel(s) of one chunk (hamming_decode on the device)
  T_PR   D2H copy of one chunk's data + syndrome bytes
  SDT    n_streams = 1: the chunks' PS, DKE, PR strictly in sequence
         -> predicted N (T_PS + T_DKE + T_PR)
  ADT    n_streams = 3: PS / DKE / PR of different chunks overlap (separate
         copy engines each way) -> predicted by the three-stage pipeline
         (T_PS + T_DKE + T_PR) + (N - 1) max(T_PS, T_DKE, T_PR),
         which is the paper's T_PS + N T_DKE + T_PR when T_DKE dominates;
         here the link dominates (T_PS + T_PR >> T_DKE, the paper's own regime
         P:L131), so the speedup tends to (T_PS + T_DKE + T_PR) / max(...) ~ 2,
         not to N.

Stage times are medians of CUDA-event-timed single stages on one stream;
makespans are wall clock around the synchronous call (median of 5).

python tools/adt_eq1.py [--out profiles/r02_adt_eq1.md]"""
import argparse
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_6862_b200 as ham  # noqa: E402


def stage_times(m, chunk, reps=7):
    """(T_PS, T_DKE, T_PR) in seconds for one chunk of `chunk` codewords."""
    n, k = ham.code_nk(m)
    rx_d = ham.channel_generate(m, 3, 0, chunk, p=0.1)
    rx_h = torch.empty(ham.coded_bytes(m, chunk), dtype=torch.uint8, pin_memory=True)
    rx_h.copy_(rx_d[: rx_h.numel()])
    d_d = torch.empty(ham.data_bytes(m, chunk), dtype=torch.uint8, device="cuda")
    s_d = torch.empty(chunk, dtype=torch.uint8, device="cuda")
    c_d = torch.empty(1, dtype=torch.int64, device="cuda")
    d_h = torch.empty_like(d_d, device="cpu").pin_memory()
    s_h = torch.empty_like(s_d, device="cpu").pin_memory()
    st = torch.cuda.Stream()
    out = {"ps": [], "dke": [], "pr": []}
    with torch.cuda.stream(st):
        for _ in range(reps):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            e[0].record(st)
            rx_d[: rx_h.numel()].copy_(rx_h, non_blocking=True)
            e[1].record(st)
            ham.decode(m, rx_d, chunk, data_out=d_d, syndromes=s_d, corrected=c_d, stream=st)
            e[2].record(st)
            d_h.copy_(d_d, non_blocking=True)
            s_h.copy_(s_d, non_blocking=True)
            e[3].record(st)
            st.synchronize()
            out["ps"].append(e[0].elapsed_time(e[1]) / 1e3)
            out["dke"].append(e[1].elapsed_time(e[2]) / 1e3)
            out["pr"].append(e[2].elapsed_time(e[3]) / 1e3)
    return tuple(statistics.median(out[x][1:]) for x in ("ps", "dke", "pr"))


def makespan(m, N, chunk, streams, reps=5):
    rx_d = ham.channel_generate(m, 5, 0, N, p=0.1)
    rx_h = torch.empty(ham.coded_bytes(m, N), dtype=torch.uint8, pin_memory=True)
    rx_h.copy_(rx_d[: rx_h.numel()])
    del rx_d
    d_h = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, pin_memory=True)
    s_h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    ws = torch.empty(ham.host_workspace_bytes(m, chunk, streams, True), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    ham.decode_host(m, rx_h, N, d_h, s_h, ws, chunk_codewords=chunk, n_streams=streams)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        ham.decode_host(m, rx_h, N, d_h, s_h, ws, chunk_codewords=chunk, n_streams=streams)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


def model(m, chunk, n_chunks):
    """One row: measured stages, predicted and measured SDT / ADT makespans."""
    tps, tdke, tpr = stage_times(m, chunk)
    N = chunk * n_chunks
    sdt_pred = n_chunks * (tps + tdke + tpr)
    adt_pred = (tps + tdke + tpr) + (n_chunks - 1) * max(tps, tdke, tpr)
    sdt = makespan(m, N, chunk, 1)
    adt = makespan(m, N, chunk, 3)
    return dict(m=m, chunk=chunk, n_chunks=n_chunks, t_ps=tps, t_dke=tdke, t_pr=tpr, sdt_pred=sdt_pred, sdt=sdt,
                adt_pred=adt_pred, adt=adt, speedup_pred=sdt_pred / adt_pred, speedup=sdt / adt,
                paper_adt=tps + n_chunks * tdke + tpr)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for m, chunk, nc in ((6, 1 << 22, 16), (6, 1 << 24, 8), (5, 1 << 23, 16), (4, 1 << 24, 16), (3, 1 << 25, 8)):
        r = model(m, chunk, nc)
        rows.append(r)
        print({k: (round(v * 1e3, 3) if isinstance(v, float) and k.startswith(("t_", "sdt", "adt", "paper"))
                   else round(v, 3) if isinstance(v, float) else v) for k, v in r.items()}, flush=True)
    lines = ["# Eq. 1 (P:L115-132) on one B200: SDT vs ADT through hamming_decode_host", "",
             "Stage times per chunk (CUDA events, median of 6), makespans (wall clock around the synchronous "
             "call, median of 5), predictions from the measured stages: SDT = N (T_PS + T_DKE + T_PR); "
             "ADT = (T_PS + T_DKE + T_PR) + (N - 1) max(T_PS, T_DKE, T_PR) (S:L384). 'paper ADT' is the "
             "paper's T_PS + N T_DKE + T_PR, which assumes the kernel dominates -- it does not here.", "",
             "| code | chunk (cw) | N chunks | T_PS ms | T_DKE ms | T_PR ms | SDT pred ms | SDT meas ms | ADT pred ms "
             "| ADT meas ms | paper ADT ms | speedup pred | speedup meas |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        n = 2 ** r["m"] - 1
        lines.append(f"| ({n},{n - r['m']}) | {r['chunk']} | {r['n_chunks']} | {r['t_ps'] * 1e3:.3f} | "
                     f"{r['t_dke'] * 1e3:.3f} | {r['t_pr'] * 1e3:.3f} | {r['sdt_pred'] * 1e3:.2f} | {r['sdt'] * 1e3:.2f} | "
                     f"{r['adt_pred'] * 1e3:.2f} | {r['adt'] * 1e3:.2f} | {r['paper_adt'] * 1e3:.2f} | "
                     f"{r['speedup_pred']:.3f} | {r['speedup']:.3f} |")
    text = "\n".join(lines) + "\n"
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)


if __name__ == "__main__":
    main()
