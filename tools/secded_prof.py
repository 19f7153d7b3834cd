import sys, torch
sys.path.insert(0, '.')
import paper_1412_6862_b200 as ham
m = 6; N = (256 << 20) * 8 // 64
rx = ham.channel_generate_secded(m, 1, 0, N, p=0.1, q2=0.1)
for _ in range(3): res = ham.decode_secded(m, rx, N)
torch.cuda.synchronize()
