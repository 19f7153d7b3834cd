"""Zero-copy experiment: hamming_decode's tile kernel given PINNED HOST pointers (UVA: the SMs'
TMA reads the packet over PCIe and writes data and syndromes back over PCIe, no DMA stages) vs the
chunked H2D / decode / D2H pipeline (hamming_decode_host), same 8 GiB (63,57) packet, wall clock.
Outputs of the two are compared byte for byte.  python tools/zero_copy_probe.py [GiB]"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402
from paper_1412_6862_b200 import _lib  # noqa: E402

gib = float(sys.argv[1]) if len(sys.argv) > 1 else 8.0
m = 6
n, k = ham.code_nk(m)
N = int(gib * (1 << 30) * 8) // n // 1024 * 1024
rx_d = ham.channel_generate(m, 1, 0, N, p=0.1)
rx_h = torch.empty(ham.coded_bytes(m, N), dtype=torch.uint8, pin_memory=True)
rx_h.copy_(rx_d[: rx_h.numel()])
del rx_d
data_h = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, pin_memory=True)
syn_h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
data_z = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, pin_memory=True)
syn_z = torch.empty(N, dtype=torch.uint8, pin_memory=True)
chunk = 1 << 24
ws = torch.empty(ham.host_workspace_bytes(m, chunk, 3, True), dtype=torch.uint8, device="cuda")
cnt_d = torch.zeros(1, dtype=torch.int64, device="cuda")
L = _lib.lib()
st = torch.cuda.current_stream().cuda_stream


def pipeline():
    return ham.decode_host(m, rx_h, N, data_h, syn_h, ws, chunk_codewords=chunk, n_streams=3)


def zero_copy():
    rc = L.hamming_decode(m, ctypes.c_void_p(rx_h.data_ptr()), ctypes.c_uint64(N), ctypes.c_void_p(data_z.data_ptr()),
                          ctypes.c_void_p(syn_z.data_ptr()), ctypes.c_void_p(cnt_d.data_ptr()), ctypes.c_void_p(st))
    assert rc == 0, rc
    c = int(cnt_d.item())  # the count back to the host (synchronises)
    return c


for name, fn in (("pipeline (H2D/decode/D2H, 3 streams)", pipeline), ("zero-copy (kernel on pinned host memory)", zero_copy)):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = min(ts)
    print(f"{name}: {t * 1e3:.1f} ms, {n * N / t / 1e9:.1f} coded Gbit/s, H2D {ham.coded_bytes(m, N) / t / 1e9:.1f} GB/s",
          flush=True)
print("outputs equal:", bool(torch.equal(data_h, data_z)) and bool(torch.equal(syn_h, syn_z)), flush=True)


# hybrid: the packet goes H2D by DMA in chunks (3 streams), the decode kernel writes data and syndromes
# straight into pinned host memory (no device output staging, no D2H DMA)
nst = 3
bufs = [torch.empty(ham.coded_bytes(m, chunk) + 64, dtype=torch.uint8, device="cuda") for _ in range(nst)]
streams = [torch.cuda.Stream() for _ in range(nst)]
cnts = torch.zeros(max(1, (N + chunk - 1) // chunk), dtype=torch.int64, device="cuda")
data_y = torch.empty(data_z.numel(), dtype=torch.uint8, pin_memory=True)
syn_y = torch.empty(syn_z.numel(), dtype=torch.uint8, pin_memory=True)


def hybrid():
    cur = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(cur)
    for i, c0 in enumerate(range(0, N, chunk)):
        nc = min(chunk, N - c0)
        s = streams[i % nst]
        b0 = c0 * n // 8
        with torch.cuda.stream(s):
            bufs[i % nst][: ham.coded_bytes(m, nc)].copy_(rx_h[b0:b0 + ham.coded_bytes(m, nc)], non_blocking=True)
            rc = L.hamming_decode(m, ctypes.c_void_p(bufs[i % nst].data_ptr()), ctypes.c_uint64(nc),
                                  ctypes.c_void_p(data_y.data_ptr() + c0 * k // 8),
                                  ctypes.c_void_p(syn_y.data_ptr() + c0), ctypes.c_void_p(cnts[i:].data_ptr()),
                                  ctypes.c_void_p(s.cuda_stream))
            assert rc == 0, (rc, i, L.hamming_last_error())
    for s in streams:
        cur.wait_stream(s)
    return int(cnts.sum().item())


hybrid()
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    hybrid()
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
t = min(ts)
print(f"hybrid (H2D DMA, kernel writes host memory): {t * 1e3:.1f} ms, {n * N / t / 1e9:.1f} coded Gbit/s", flush=True)
print("hybrid outputs equal:", bool(torch.equal(data_h, data_y)) and bool(torch.equal(syn_h, syn_y)), flush=True)
