"""Steady-state power and bandwidth of the decode kernels vs a plain copy of
the same byte volume: each kernel runs back to back for ~3 s while
nvidia-smi samples power.draw and clocks.sm every 50 ms.

With a probe build (python tools/power_probe.py --probe: builds
tune_libs/probe.so with -DHAM_PROBE and points HAMMING_LIB at it) it also runs
the (63,57) tile pipeline with the decode taken out -- TMA in/out only
(ProbeTmaOp), and TMA plus the lane's shared-memory loads/stores (ProbeLdsOp)
-- so the decode's power splits into the round trip and the arithmetic.
python tools/power_probe.py [--probe] [--only6]"""
import ctypes
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
PROBE = "--probe" in sys.argv
ONLY6 = "--only6" in sys.argv
if PROBE and "HAMMING_LIB" not in os.environ:
    from paper_1412_6862_b200 import build as _b
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    os.makedirs(os.path.join(root, "tune_libs"), exist_ok=True)
    os.environ["HAMMING_LIB"] = _b.build(force=True, out=os.path.join(root, "tune_libs", "probe.so"),
                                         defines=["HAM_PROBE"])
import paper_1412_6862_b200 as ham  # noqa: E402
from paper_1412_6862_b200 import _lib  # noqa: E402


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm,clocks.mem", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append([float(x) for x in line.split(",")])
    p.terminate()


def run(name, fn, nbytes, seconds=3.0):
    fn()
    torch.cuda.synchronize()
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, rows))
    th.start()
    time.sleep(0.3)
    t0 = time.time()
    n = 0
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < seconds:
        for _ in range(10):
            fn()
        n += 10
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = s.elapsed_time(e) / n
    late = rows[len(rows) // 2:] or rows
    pw = sum(r[0] for r in late) / len(late)
    sm = sum(r[1] for r in late) / len(late)
    print(f"{name:28s} {nbytes / ms / 1e6:8.0f} GB/s  power {pw:6.0f} W  sm {sm:6.0f} MHz  "
          f"({nbytes / ms / 1e6 / pw:.2f} GB/s per W)", flush=True)


G = 8 << 30
a = torch.empty(G // 2, dtype=torch.uint8, device="cuda")
b = torch.empty(G // 2, dtype=torch.uint8, device="cuda")
if "--no-copy" not in sys.argv:
    run("copy 4 GiB -> 4 GiB", lambda: b.copy_(a), G)
del a, b
if PROBE:
    L = _lib.lib()
    L.hamming_probe_tiles.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p]
    N = (4 << 30) * 8 // 63 // 1024 * 1024
    rx = torch.empty(ham.coded_bytes(6, N), dtype=torch.uint8, device="cuda").random_(0, 256)
    out = torch.empty(ham.coded_bytes(6, N), dtype=torch.uint8, device="cuda")  # kinds 3, 4 write ib bytes
    syn = torch.empty(N, dtype=torch.uint8, device="cuda")
    cnt = torch.empty(1, dtype=torch.int64, device="cuda")
    alg = ham.coded_bytes(6, N) + ham.data_bytes(6, N) + N
    kinds = ((0, "probe TMA only (63,57) tiles"), (1, "probe TMA + LDS/STS"), (2, "probe TMA only, no syndromes"),
             (3, "probe TMA copy (63-word tiles)"), (4, "probe LDG/STG copy"))
    for kind, nm in kinds:
        def fn(kind=kind):
            rc = L.hamming_probe_tiles(kind, rx.data_ptr(), N, out.data_ptr(), syn.data_ptr(), cnt.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream)
            assert rc == 0, rc
        # kind 2 writes no syndrome bytes; kinds 3, 4 read and write the coded bytes
        run(nm, fn, alg - N if kind == 2 else (2 * ham.coded_bytes(6, N) if kind >= 3 else alg))
    del rx, out, syn
    torch.cuda.empty_cache()
for m in ((6,) if ONLY6 else (6, 5, 4, 3)):
    n, k = ham.code_nk(m)
    N = (4 << 30) * 8 // n // 1024 * 1024
    rx = ham.channel_generate(m, 1, 0, N, p=0.1)
    res = ham.decode(m, rx, N)
    alg = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
    run(f"decode m={m} 4 GiB", lambda: ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes,
                                                  corrected=res.corrected), alg)
    del rx, res
    torch.cuda.empty_cache()
