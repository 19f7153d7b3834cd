"""Forced packet launch shapes (a -DHAM_PKT_TUNE build, HAM_PKT_W / HAM_PKT_G from the
environment) for a few (M, t): python tools/pkt_shape_sweep.py <lib.so>"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1]
cells = [(400, 5), (400, 2), (800, 6), (1200, 2), (2000, 3)]
for M, t in cells:
    for w in (4, 8, 12):
        for G in (2, 3, 4, 6, 8, 10, 12, 16, 24):
            env = dict(os.environ, HAMMING_LIB=lib, HAM_PKT_W=str(w), HAM_PKT_G=str(G))
            r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "packets_bench.py"), "--M", str(M), "--t", str(t),
                                "--reps", "3"], env=env, capture_output=True, text=True)
            line = (r.stdout.strip().splitlines() or [r.stderr.strip()[-200:]])[-1]
            print(f"w={w} G={G} {line}", flush=True)
