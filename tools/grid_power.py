"""Power, SM clock and bandwidth of the sustained (63,57) decode when its tile grid covers fewer SMs
(a -DHAM_GRID_TUNE build reads HAM_GRID_SMS at every call): python tools/grid_power.py <lib.so>.
Each row: ~3 s back to back on 4 GiB coded, nvidia-smi sampled every 50 ms (second half), plus the
first 0.5 s alone (the bench's 20-step window)."""
import os
import subprocess
import sys
import threading
import time

os.environ["HAMMING_LIB"] = sys.argv[1]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1412_6862_b200 as ham  # noqa: E402
import json  # noqa: E402

PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]


def sample(stop, rows):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=power.draw,clocks.sm", "--format=csv,noheader,nounits", "-lms", "50"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if line:
            rows.append([float(x) for x in line.split(",")])
    p.terminate()


m = 6
n, k = ham.code_nk(m)
N = (4 << 30) * 8 // n // 1024 * 1024
rx = ham.channel_generate(m, 1, 0, N, p=0.1)
res = ham.decode(m, rx, N)
alg = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
fn = lambda: ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected)  # noqa: E731
for sms in [int(x) for x in (sys.argv[2:] or ["148", "140", "132", "124", "116", "108"])]:
    os.environ["HAM_GRID_SMS"] = str(sms)
    fn()
    torch.cuda.synchronize()
    time.sleep(2.0)  # start each row from a cool board
    rows, stop = [], threading.Event()
    th = threading.Thread(target=sample, args=(stop, rows))
    th.start()
    evs = []
    t0 = time.time()
    while time.time() - t0 < 3.0:
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        evs.append((s, e))
        if len(evs) % 8 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ts = [s.elapsed_time(e) for s, e in evs]
    first = ts[: max(1, int(500 / (sum(ts) / len(ts))))]
    late = rows[len(rows) // 2:] or rows
    pw = sum(r[0] for r in late) / len(late)
    sm = sum(r[1] for r in late) / len(late)
    f_all = alg / (sum(ts) / len(ts)) / 1e6 / PEAK
    f_first = alg / (sum(first) / len(first)) / 1e6 / PEAK
    print(f"grid SMs {sms:3d} (grid {ham.last_grid_blocks()}): first 0.5 s {f_first:.3f}, 3 s {f_all:.3f} of copy peak; "
          f"power {pw:5.0f} W, sm {sm:5.0f} MHz", flush=True)
