"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every decode shape with ragged tails, encode, generate and the
host pipeline, at sizes that keep the sanitizer fast.

--initcheck: the same kernels on random received bytes written by a torch
kernel, without the workload's own torch/cudaMemcpy copies of kernel outputs
and without the host pipeline.  initcheck does not
count bytes written by TMA bulk stores (cp.async.bulk) as initialised, so a
cudaMemcpy that reads them is reported ("Uninitialized access ... by
cudaMemcpy source", 12 472 such reports with the copies in, none from a kernel);
without the copies what is left are the kernels' own accesses."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1412_6862_b200 as ham  # noqa: E402

INIT = "--initcheck" in sys.argv

for m in (2, 3, 4, 5, 6):
    for N in (1, 1023, 3 * 1024 + 77, 20_000):
        if INIT:  # written by a torch kernel (initcheck does not see TMA bulk stores as writes)
            exact = torch.randint(0, 256, (ham.coded_bytes(m, N),), dtype=torch.uint8, device="cuda")
        else:
            exact = torch.empty(ham.coded_bytes(m, N), dtype=torch.uint8, device="cuda")
            ham.channel_generate(m, 7, 0, N, p=0.3, q2=0.3, rx_out=exact)  # exactly the coded bytes
        res = ham.decode(m, exact, N)
        ham.decode(m, exact, N, syndromes=False)
        if INIT:
            data = res.data
        else:
            data = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, device="cuda")
            data.copy_(res.data[: data.numel()])
        ham.encode(m, data, N)
        torch.cuda.synchronize()
    if INIT:
        continue
    N = 5 * 1024 + 3
    rx = ham.channel_generate(m, 9, 0, N, p=0.2).cpu()
    ws = torch.empty(ham.host_workspace_bytes(m, 2048, 2, True), dtype=torch.uint8, device="cuda")
    ham.decode_host(m, rx, N, torch.empty(ham.data_bytes(m, N), dtype=torch.uint8),
                    torch.empty(N, dtype=torch.uint8), ws, chunk_codewords=2048, n_streams=2)
# SECDED, long perfect codes, the paper's packets
for m in (3, 4, 5, 6):
    for N in (1, 3 * 1024 + 77):
        rx = ham.channel_generate_secded(m, 5, 0, N, p=0.5, q2=0.5)
        res = ham.decode_secded(m, rx, N)
        if INIT:
            data = res.data
        else:
            data = torch.empty(ham.data_bytes(m, N), dtype=torch.uint8, device="cuda")
            data.copy_(res.data[: data.numel()])
        ham.encode_secded(m, data, N)
        torch.cuda.synchronize()
for m in (7, 8):
    for N in (1, 128 * 5 + 3):
        rx = torch.randint(0, 256, (ham.coded_bytes(m, N),), dtype=torch.uint8, device="cuda")
        ham.decode(m, rx, N)
        torch.cuda.synchronize()
# packets: with head compaction (k >= 96: 400/6, 400/5, 2000/2, 1200/3, 97/8) and without (13/3,
# 71/6), several launch shapes (8, 12, 16 warps; 1..10 packets per batch), uncorrectable segments
for M, t in ((400, 6), (400, 5), (2000, 2), (1200, 3), (97, 8), (13, 3), (71, 6)):
    rx, _ = ham.packet_channel_generate(M, t, 1, 0, 37, p=1.0)
    ham.decode_packets(M, t, rx, 37)
    noise = torch.randint(0, 256, rx.shape, dtype=torch.uint8, device="cuda")
    ham.decode_packets(M, t, noise, 37)
    torch.cuda.synchronize()
print("sanitize workload done")
