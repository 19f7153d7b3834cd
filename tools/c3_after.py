"""Does the C3 per-call rate depend on what ran before?  (a) after a 100 GiB
allocation was freed (allocator / TLB state), (b) right after ~10 s of
back-to-back 64 GiB-class decode load (power / thermal state).  Runs
tools/c3_probe.py's measurement after each.  python tools/c3_after.py"""
import os
import runpy
import subprocess
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1412_6862_b200 as ham  # noqa: E402


def smi():
    q = "clocks.sm,power.draw.instant,temperature.gpu,clocks_event_reasons.sw_power_cap"
    return subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader"], capture_output=True,
                          text=True).stdout.strip()


mode = sys.argv[1] if len(sys.argv) > 1 else "big"
if mode == "big":
    x = torch.empty(100 << 30, dtype=torch.uint8, device="cuda")
    x.fill_(1)
    del x
    torch.cuda.empty_cache()
    print("after a freed 100 GiB allocation:", smi(), flush=True)
else:
    m, N = 6, (48 << 30) * 8 // 63
    rx = ham.channel_generate(m, 1, 0, N, p=0.1)
    res = ham.decode(m, rx, N)
    t0 = time.time()
    while time.time() - t0 < 10:
        for _ in range(20):
            ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes, corrected=res.corrected)
        torch.cuda.synchronize()
    print("after 10 s of (63,57) decode load:", smi(), flush=True)
    del rx, res
    torch.cuda.empty_cache()
sys.argv = [sys.argv[0], "3", "4", "6"]
runpy.run_path(os.path.join(ROOT, "tools", "c3_probe.py"), run_name="__main__")
print("end:", smi(), flush=True)
