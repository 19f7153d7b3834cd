"""Steady-state power and bandwidth of the decode kernels vs a plain copy of
the same byte volume: each kernel runs back to back for ~3 s while
nvidia-smi samples power.draw and clocks.sm every 50 ms."""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402


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
run("copy 4 GiB -> 4 GiB", lambda: b.copy_(a), G)
del a, b
for m in (6, 5, 4, 3):
    n, k = ham.code_nk(m)
    N = (4 << 30) * 8 // n // 1024 * 1024
    rx = ham.channel_generate(m, 1, 0, N, p=0.1)
    res = ham.decode(m, rx, N)
    alg = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
    run(f"decode m={m} 4 GiB", lambda: ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes,
                                                  corrected=res.corrected), alg)
    del rx, res
    torch.cuda.empty_cache()
