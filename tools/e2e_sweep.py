"""hamming_decode_host (the e2e path, P:L113-132 ADT) on an 8 GiB (63,57) host packet:
wall time per call over chunk sizes and stream counts.  python tools/e2e_sweep.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

m, n = 6, 63
N = (8 << 30) * 8 // n // 1024 * 1024
rx_d = ham.channel_generate(m, 1, 0, N, p=0.1)
rx_h = torch.empty(ham.coded_bytes(m, N), dtype=torch.uint8, pin_memory=True)
rx_h.copy_(rx_d[: rx_h.numel()])
del rx_d
data_h = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, pin_memory=True)
syn_h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
for chunk in (1 << 22, 1 << 23, 1 << 24, 1 << 25):
    for ns in (2, 3, 4):
        ws = torch.empty(ham.host_workspace_bytes(m, chunk, ns, True), dtype=torch.uint8, device="cuda")
        ham.decode_host(m, rx_h, N, data_h, syn_h, ws, chunk_codewords=chunk, n_streams=ns)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            ham.decode_host(m, rx_h, N, data_h, syn_h, ws, chunk_codewords=chunk, n_streams=ns)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"chunk {chunk} streams {ns}: {t * 1e3:.1f} ms, {n * N / t / 1e9:.0f} coded Gbit/s, "
              f"H2D {ham.coded_bytes(m, N) / t / 1e9:.1f} GB/s", flush=True)
        del ws
        torch.cuda.empty_cache()
