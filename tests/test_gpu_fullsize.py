"""Full-size parity (-m gpu) at BASELINE.json's configurations, in the launch
configuration bench.py times: the GPU generates the packet on the device
(its generator is checked byte-for-byte against the oracle's in
test_gpu_parity.py), decodes it with the same call bench.py times, and the
oracle -- regenerating each sampled window from the seed on its own --
decodes sampled windows (first, last and seeded random ones) that are
compared bit for bit.  The count is checked against properties that hold at
any size."""
import os

import numpy as np
import pytest
import torch

import paper_1412_6862_b200 as ham

pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)))


def check_windows(oracle, m, seed, N, p, q2, res, n_windows=24, w=1 << 14):
    n, k = ham.code_nk(m)
    rng = np.random.default_rng(seed)
    starts = {0, max(0, (N - w) // 8 * 8)}
    while len(starts) < n_windows + 2 and N > w:
        starts.add(int(rng.integers(0, N - w)) // 8 * 8)
    for c0 in sorted(starts):
        cnt = min(w, N - c0)
        rx, _, _ = oracle.generate(m, seed, c0, cnt, p=p, q2=q2, threads=THREADS)
        wd, ws, wc = oracle.decode_mt(m, rx, cnt, THREADS)
        db = ham.data_bytes(m, cnt)
        got_d = res.data[c0 * k // 8: c0 * k // 8 + db].cpu().numpy()
        if (cnt * k) % 8 and c0 + cnt < N:  # window ends mid-byte inside the stream: compare whole bytes only
            got_d, wd = got_d[:-1], wd[:-1]
        assert np.array_equal(got_d, wd), (m, N, c0)
        got_s = res.syndromes[c0: c0 + cnt].cpu().numpy()
        assert np.array_equal(got_s, ws), (m, N, c0)


def decode_config(oracle, m, N, seed, p, q2):
    rx = ham.channel_generate(m, seed, 0, N, p=p, q2=q2)
    res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    check_windows(oracle, m, seed, N, p, q2, res)
    corrected = int(res.corrected.item())
    nonzero = sum(int(torch.count_nonzero(res.syndromes[i:min(N, i + (1 << 30))]).item())
                  for i in range(0, N, 1 << 30))
    assert corrected == nonzero
    # every error event gives a nonzero syndrome (1 or 2 flips, p1 != p2)
    sd = np.sqrt(N * p * (1 - p)) if 0 < p < 1 else 0
    assert abs(corrected - N * p) <= 6 * sd + 1, (corrected, N * p)
    # the pad bits of the data stream are zero
    tail_bits = (N * ham.code_nk(m)[1]) % 8
    if tail_bits:
        assert int(res.data[ham.data_bytes(m, N) - 1].item()) >> tail_bits == 0
    del rx, res
    torch.cuda.empty_cache()


def test_c1_one_4kb_packet(oracle):
    """configs[0]: (7,4), one 4 KB packet (4681 codewords), p = 0.1 -- in full."""
    m, N, seed = 3, 4681, 0x14126862
    rx_np, sent, err = oracle.generate(m, seed, 0, N, p=0.1, want_sent=True, want_err=True)
    rx = ham.channel_generate(m, seed, 0, N, p=0.1)
    torch.cuda.synchronize()
    assert np.array_equal(rx.cpu().numpy()[: rx_np.size], rx_np)
    res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    wd, ws, wc = oracle.decode(m, rx_np, N)
    assert np.array_equal(res.data.cpu().numpy()[: wd.size], wd)
    assert np.array_equal(res.syndromes.cpu().numpy()[:N], ws)
    assert res.corrected.item() == wc == int((err.reshape(N, 2)[:, 0] > 0).sum())
    assert np.array_equal(wd, sent)


@pytest.mark.parametrize("size", [1 << 10, 400, 2000, 1 << 16, 1 << 20, 1 << 26])
def test_c2_packet_size_sweep(oracle, size):
    """configs[1]: (15,11) packets of 1 KB .. 64 MB coded bytes."""
    m = 4
    N = size * 8 // 15
    decode_config(oracle, m, N, 0x14126862 ^ size, 0.1, 0.0)


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_c3_code_length_sweep_256mb(oracle, m):
    """configs[2]: 256 MiB bit-packed packets for m = 3..6."""
    n, _ = ham.code_nk(m)
    N = (256 << 20) * 8 // n
    decode_config(oracle, m, N, 0x14126862 ^ (m << 4), 0.1, 0.0)


@pytest.mark.parametrize("p", [0.0, 1e-3, 0.1, 0.5, 1.0])
def test_c4_error_sweep_1gb(oracle, p):
    """configs[3]: (31,26), 1 GiB, p in [0, 1] with q2 = 0.25 (2-bit events:
    the GPU must make the oracle's miscorrection)."""
    m = 5
    N = (1 << 30) * 8 // 31
    decode_config(oracle, m, N, 0x14126862 ^ int(p * 1000), p, 0.25)


def test_c5_bench_workload_64gb(oracle):
    """configs[4] at one GPU: (63,57), 2^39 coded bits (64 GiB), the exact
    call bench.py times; sampled windows against the oracle."""
    m = 6
    N = (1 << 39) // 63
    free, _ = torch.cuda.mem_get_info()
    need = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
    if free < need + (2 << 30):
        pytest.skip(f"needs {need / 2**30:.0f} GiB free device memory, have {free / 2**30:.0f}")
    decode_config(oracle, m, N, 0x14126862 ^ 5, 0.1, 0.0)
