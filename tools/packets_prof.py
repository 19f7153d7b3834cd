"""One hamming_decode_packets launch for ncu: python tools/packets_prof.py M t [P]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

M, t = int(sys.argv[1]), int(sys.argv[2])
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 19
rx, _ = ham.packet_channel_generate(M, t, 3, 0, P, p=1.0)
out = torch.empty(P * M, dtype=torch.uint8, device="cuda")
for _ in range(2):
    ham.decode_packets(M, t, rx, P, msg_out=out)
torch.cuda.synchronize()
