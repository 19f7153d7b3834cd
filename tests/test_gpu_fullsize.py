"""Full-size parity (-m gpu) at BASELINE.json's configurations, in the launch
configuration bench.py times: the GPU generates the packet on the device and
decodes it with the very call bench.py times; the CPU oracle regenerates the
same packet from the seed on its own (host threads over disjoint ranges, the
per-codeword code plain C) and decodes it.

  * C1, C2 (every size), C3 (every m; m = 3, 4 also with 2-bit events) and C4
    (every p of the sweep): the WHOLE output -- received stream, data stream,
    every syndrome byte and the exact count -- is compared (SURVEY.md 8(c),
    8(d); "decode mismatch -> hard failure").
  * C5 (64 GiB, larger than the host oracle can decode in a test): the
    survey's stratified sample -- the first and the last 2^20 codewords plus
    64 seeded random 2^20-codeword windows -- and the exact count against the
    oracle's own count of the channel's error events over all 8.7e9
    codewords (q2 = 0: every event is one flip, whose syndrome is nonzero).
"""
import os

import numpy as np
import pytest
import torch

import paper_1412_6862_b200 as ham

pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)))
SEED = 0x14126862


def assert_bytes_equal(got: np.ndarray, want: np.ndarray, what: str):
    assert got.shape == want.shape, (what, got.shape, want.shape)
    if not np.array_equal(got, want):
        bad = np.flatnonzero(got != want)
        raise AssertionError(f"{what}: {bad.size} bytes differ, first at {bad[:8].tolist()}: "
                             f"{got[bad[:8]].tolist()} vs {want[bad[:8]].tolist()}")


def full_check(oracle, m, N, seed, p, q2):
    """The whole packet: GPU generator + the bench's decode call, against the
    oracle's generator + decoder, every byte and the exact count."""
    rx = ham.channel_generate(m, seed, 0, N, p=p, q2=q2)
    res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    got_rx = rx[: ham.coded_bytes(m, N)].cpu().numpy()
    got_d = res.data[: ham.data_bytes(m, N)].cpu().numpy()
    got_s = res.syndromes[:N].cpu().numpy()
    got_c = int(res.corrected.item())
    del rx, res
    torch.cuda.empty_cache()
    want_rx, _, _ = oracle.generate(m, seed, 0, N, p=p, q2=q2, threads=THREADS)
    assert_bytes_equal(got_rx, want_rx, f"m={m} N={N} received stream")
    del got_rx
    wd, ws, wc = oracle.decode_mt(m, want_rx, N, THREADS)
    assert_bytes_equal(got_d, wd, f"m={m} N={N} p={p} q2={q2} data")
    assert_bytes_equal(got_s, ws, f"m={m} N={N} p={p} q2={q2} syndromes")
    assert got_c == wc, (m, N, p, q2, got_c, wc)
    ev, w2 = oracle.count_events(seed, 0, N, p=p, q2=q2, threads=THREADS)
    # every event gives a nonzero syndrome -- one flip at p1, or two at p1 != p2 (s = p1 ^ p2,
    # a miscorrection, counted too: reading R10) -- so the count is the number of events
    assert wc == ev, (wc, ev, w2)
    return wc


def test_c1_one_4kb_packet(oracle):
    """configs[0]: (7,4), one 4 KB packet (4681 codewords), p = 0.1, against the
    sent data as well (single flips are all corrected)."""
    m, N = 3, 4681
    rx_np, sent, err = oracle.generate(m, SEED, 0, N, p=0.1, want_sent=True, want_err=True)
    rx = ham.channel_generate(m, SEED, 0, N, p=0.1)
    torch.cuda.synchronize()
    assert np.array_equal(rx.cpu().numpy()[: rx_np.size], rx_np)
    res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    wd, ws, wc = oracle.decode(m, rx_np, N)
    assert np.array_equal(res.data.cpu().numpy()[: wd.size], wd)
    assert np.array_equal(res.syndromes.cpu().numpy()[:N], ws)
    assert res.corrected.item() == wc == int((err.reshape(N, 2)[:, 0] > 0).sum())
    assert np.array_equal(wd, sent)


C2_SIZES = [1 << e for e in range(10, 27)] + [400, 800, 1200, 1600, 2000]


@pytest.mark.parametrize("size", C2_SIZES)
def test_c2_packet_size_sweep(oracle, size):
    """configs[1]: (15,11) packets of 1 KB .. 64 MB coded bytes (17 powers of
    two) plus the paper's 400..2000-byte packets, each in full."""
    m = 4
    full_check(oracle, m, size * 8 // 15, SEED ^ size, 0.1, 0.0)


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_c3_code_length_sweep_256mb(oracle, m):
    """configs[2]: 256 MiB bit-packed packets for m = 3..6, in full."""
    n, _ = ham.code_nk(m)
    full_check(oracle, m, (256 << 20) * 8 // n, SEED ^ (m << 4), 0.1, 0.0)


@pytest.mark.parametrize("m", [3, 4])
def test_c3_table_decoders_with_double_errors(oracle, m):
    """configs[2] for the (7,4) / (15,11) table decoders that serve every
    call above the small-call limit (2 MiB coded), with 2-bit events
    (miscorrections) -- in full."""
    n, _ = ham.code_nk(m)
    full_check(oracle, m, (256 << 20) * 8 // n, SEED ^ (m << 4) ^ 0x2B, 0.25, 0.25)


C4_P = [0.0, 1e-3, 1e-2, 0.1, 0.25, 0.5, 0.75, 1.0]


@pytest.mark.parametrize("p", C4_P)
def test_c4_error_sweep_1gb(oracle, p):
    """configs[3]: (31,26), 1 GiB, every p of the sweep with q2 = 0.25 (2-bit
    events: the GPU must make the oracle's miscorrection) -- in full."""
    m = 5
    N = (1 << 30) * 8 // 31
    wc = full_check(oracle, m, N, SEED ^ int(p * 1000), p, 0.25)
    if p == 0.0:
        assert wc == 0
    if p == 1.0:
        assert wc == N


@pytest.mark.parametrize("q2", [0.0, 1.0])
def test_c4_corners(oracle, q2):
    """configs[3] corners at p = 1: the paper regime (one error in every
    codeword, all corrected) and every codeword a 2-bit event (all
    miscorrected); 2^24 codewords each."""
    m, N = 5, 1 << 24
    assert full_check(oracle, m, N, SEED ^ 0xC4 ^ int(q2), 1.0, q2) == N


def test_c5_bench_workload_64gb(oracle):
    """configs[4] at one GPU: (63,57), 2^39 coded bits (64 GiB), the exact
    call bench.py times.  Stratified sample (first and last 2^20 codewords +
    64 seeded random 2^20 windows) against the oracle, every byte of each
    window; the count exactly against the oracle's event count."""
    m, p, q2 = 6, 0.1, 0.0
    n, k = ham.code_nk(m)
    N = (1 << 39) // n
    seed = SEED ^ 5
    free, _ = torch.cuda.mem_get_info()
    need = ham.coded_bytes(m, N) + ham.data_bytes(m, N) + N
    if free < need + (2 << 30):
        pytest.skip(f"needs {need / 2**30:.0f} GiB free device memory, have {free / 2**30:.0f}")
    rx = ham.channel_generate(m, seed, 0, N, p=p, q2=q2)
    res = ham.decode(m, rx, N)
    torch.cuda.synchronize()
    w = 1 << 20
    rng = np.random.default_rng(seed)
    last = (N - w) // 8 * 8
    starts = {0, last}
    while len(starts) < 66:
        starts.add(int(rng.integers(0, N - w)) // 8 * 8)
    for c0 in sorted(starts):
        cnt = N - c0 if c0 == last else w  # the last window runs to the end of the packet
        want_rx, _, _ = oracle.generate(m, seed, c0, cnt, p=p, q2=q2, threads=THREADS)
        got_rx = rx[c0 * n // 8: c0 * n // 8 + want_rx.size].cpu().numpy()
        assert_bytes_equal(got_rx, want_rx, f"C5 received window at {c0}")
        wd, ws, _ = oracle.decode_mt(m, want_rx, cnt, THREADS)
        got_d = res.data[c0 * k // 8: c0 * k // 8 + wd.size].cpu().numpy()
        assert_bytes_equal(got_d, wd, f"C5 data window at {c0}")
        assert_bytes_equal(res.syndromes[c0: c0 + cnt].cpu().numpy(), ws, f"C5 syndrome window at {c0}")
    ev, _ = oracle.count_events(seed, 0, N, p=p, q2=q2, threads=THREADS)
    assert int(res.corrected.item()) == ev
    del rx, res
    torch.cuda.empty_cache()
