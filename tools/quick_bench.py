import torch, time, sys
sys.path.insert(0, '.')
import paper_1412_6862_b200 as ham
for m in (3,4,5,6):
    n,k = ham.code_nk(m)
    N = (1<<31)*8//n//1024*1024   # 2 GiB coded
    rx = ham.channel_generate(m, 1, 0, N, p=0.1)
    res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    for syn in (True, False):
        ts=[]
        for i in range(8):
            s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
            s.record(); ham.decode(m, rx, N, data_out=res.data, syndromes=res.syndromes if syn else False, corrected=res.corrected); e.record(); torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        t=min(ts)/1e3
        by = ham.coded_bytes(m,N)+ham.data_bytes(m,N)+(N if syn else 0)
        print(f"m={m} syn={syn} N={N} t={t*1e3:.3f}ms  {n*N/t/1e9:.0f} Gbit/s  {by/t/1e9:.0f} GB/s grid={ham.last_grid_blocks()}", flush=True)
    del rx, res; torch.cuda.empty_cache()
