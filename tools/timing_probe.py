"""Where a 256 MiB decode spends its fixed time: per-CTA %globaltimer stamps
from a HAM_TIMING build (entry, first tile ready, loop done, stores drained).
    python -m paper_1412_6862_b200.build -o build/tune/timing.so -D HAM_TIMING
    HAMMING_LIB=build/tune/timing.so python tools/timing_probe.py [m] [MiB]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402
from paper_1412_6862_b200 import _lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
mib = float(sys.argv[2]) if len(sys.argv) > 2 else 256
n, k = ham.code_nk(m)
N = int(mib * (1 << 20) * 8) // n // 1024 * 1024
rx = ham.channel_generate(m, 1, 0, N, p=0.1)
res = ham.decode(m, rx, N)
lib = _lib.lib()
buf = (ctypes.c_ulonglong * 4096)()
for rep in range(4):
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected)
    e.record()
    torch.cuda.synchronize()
    lib.hamming_debug_timing(buf, 4096)
    g = ham.last_grid_blocks()
    a = np.array(buf[: 4 * g], dtype=np.uint64).reshape(g, 4).astype(np.int64)
    t0 = a[:, 0].min()
    r = (a - t0) / 1e3
    print(f"rep {rep}: event {s.elapsed_time(e) * 1e3:.1f} us, CTAs {g}: start {r[:, 0].min():.1f}..{r[:, 0].max():.1f}"
          f" first-tile {r[:, 1].min():.1f}..{np.median(r[:, 1]):.1f}..{r[:, 1].max():.1f}"
          f" loop-done {r[:, 2].min():.1f}..{np.median(r[:, 2]):.1f}..{r[:, 2].max():.1f}"
          f" drained {r[:, 3].min():.1f}..{r[:, 3].max():.1f} us", flush=True)
