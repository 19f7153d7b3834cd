"""Three SECDED decodes of 256 MiB coded for ncu: python tools/secded_prof.py [m]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 6
N = (256 << 20) * 8 // (1 << m)
rx = ham.channel_generate_secded(m, 1, 0, N, p=0.1, q2=0.1)
for _ in range(3):
    res = ham.decode_secded(m, rx, N)
torch.cuda.synchronize()
