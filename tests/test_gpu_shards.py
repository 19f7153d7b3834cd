"""Multi-GPU sharding through the CUDA path (-m gpu; P:L200
"the GPU deals with the segments in parallel"; S:L329 workers 1, 2, 4, 8):
the packet is cut into R = 2, 4, 8 codeword-range shards exactly as each
rank of bench.py / dist.decode_sharded cuts it (shard_range), every shard is
decoded by its own hamming_decode call on pointer offsets into the shared
buffers, and the rank-order concatenation of data and syndromes plus the
summed counts must equal the single call (itself checked against the oracle).
Also runs bench.py's N > 1 code path end to end (two ranks sharing this GPU
over gloo): self-relaunch, shards, max-over-ranks timing, JSON line."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import paper_1412_6862_b200 as ham

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
THREADS = max(1, len(os.sched_getaffinity(0)))


def _packet(m, N, seed):
    if m <= 6:
        return ham.channel_generate(m, seed, 0, N, p=0.3, q2=0.3)
    rng = np.random.default_rng(seed)
    return torch.from_numpy(rng.integers(0, 256, ham.coded_bytes(m, N), dtype=np.uint8)).cuda()


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("N", [3_000_077, 70_000])
def test_shards_concatenate_to_single_call(oracle, m, N):
    n, k = ham.code_nk(m)
    rx = _packet(m, N, 0x5A4D + m)
    full = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    fd = full.data[: ham.data_bytes(m, N)].cpu().numpy()
    fs = full.syndromes[:N].cpu().numpy()
    fc = int(full.corrected.item())
    wd, ws, wc = oracle.decode_mt(m, rx[: ham.coded_bytes(m, N)].cpu().numpy(), N, THREADS)
    assert np.array_equal(fd, wd) and np.array_equal(fs, ws) and fc == wc
    for R in (2, 4, 8):
        data = torch.full((ham.data_bytes(m, N),), 0xA5, dtype=torch.uint8, device="cuda")
        syn = torch.full((N,), 0xA5, dtype=torch.uint8, device="cuda")
        cnts = torch.zeros(R, dtype=torch.int64, device="cuda")
        for r in range(R):
            a, b = ham.shard_range(N, r, R)
            assert (a * n) % 128 == 0 and (a * k) % 128 == 0   # 16-byte aligned shard starts
            ham.decode(m, rx[a * n // 8:], b - a, data_out=data[a * k // 8:], syndromes=syn[a:],
                       corrected=cnts[r:r + 1])
        torch.cuda.synchronize()
        assert np.array_equal(data.cpu().numpy(), fd), (m, N, R)
        assert np.array_equal(syn.cpu().numpy(), fs), (m, N, R)
        assert int(cnts.sum().item()) == fc, (m, N, R)


def test_bench_two_ranks_gloo_on_one_gpu():
    """`python bench.py --gpus 2` relaunches itself as two ranks (torchrun);
    HAMMING_BENCH_BACKEND=gloo lets both share this GPU."""
    env = dict(os.environ, HAMMING_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup",
                          "3", "--config", "c3m6", "--no-e2e", "--no-cpu"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["comm"]["world_size"] == 2 and d["comm"]["ranks_reduced"] == 2
    assert d["config"]["parallelism"].startswith("dp2") and d["value"] > 0
    n = 63
    N = (256 << 20) * 8 // n
    assert d["config"]["n_codewords"] == N and d["config"]["n_codewords_per_rank"] == ham.shard_range(N, 0, 2)[1]
