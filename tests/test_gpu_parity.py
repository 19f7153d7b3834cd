"""GPU parity (-m gpu): the CUDA path through the C ABI against the CPU oracle,
bit for bit, on identical seeded packets -- data stream, syndromes and the
corrected count -- including multi-error codewords (where both must make the
same miscorrection), ragged tails, empty input and every received word of
the (7,4) and (15,11) codes."""
import os

import numpy as np
import pytest
import torch

import paper_1412_6862_b200 as ham

pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)))
SIZES = [1, 31, 32, 33, 127, 128, 129, 1023, 1024, 1025, 4681, 3 * 1024 + 17, 7 * 1024, 50_000]


def gpu(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_decode(m, rx_np, N, syndromes=True):
    res = ham.decode(m, gpu(rx_np), N, syndromes=syndromes)
    torch.cuda.synchronize()
    data = res.data.cpu().numpy()[: ham.data_bytes(m, N)]
    syn = res.syndromes.cpu().numpy()[:N] if res.syndromes is not None else None
    return data, syn, int(res.corrected.item())


def assert_same(m, N, got, want):
    d, s, c = got
    wd, ws, wc = want
    assert d.shape == wd.shape
    if not np.array_equal(d, wd):
        bad = np.nonzero(d != wd)[0][:8]
        raise AssertionError(f"m={m} N={N}: data differs at bytes {bad.tolist()}")
    if s is not None:
        if not np.array_equal(s, ws):
            bad = np.nonzero(s != ws)[0][:8]
            raise AssertionError(f"m={m} N={N}: syndromes differ at {bad.tolist()}: {s[bad]} vs {ws[bad]}")
    assert c == wc, (m, N, c, wc)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("N", SIZES)
def test_decode_matches_oracle(oracle, m, N):
    rx, _, _ = oracle.generate(m, 0x1412 + N, 0, N, p=0.5, q2=0.3)
    assert_same(m, N, gpu_decode(m, rx, N), oracle.decode(m, rx, N))


@pytest.mark.parametrize("m", [3, 6])
def test_decode_without_syndromes(oracle, m):
    N = 5000
    rx, _, _ = oracle.generate(m, 5, 0, N, p=0.2, q2=0.5)
    d, s, c = gpu_decode(m, rx, N, syndromes=False)
    wd, _, wc = oracle.decode(m, rx, N)
    assert s is None and np.array_equal(d, wd) and c == wc


@pytest.mark.parametrize("m,N", [(2, 8), (3, 128), (4, 32768)])
def test_every_received_word(oracle, m, N):
    """All 2^n received words of the code, one codeword each."""
    n = 2 ** m - 1
    words = np.arange(N, dtype=np.int64)
    bits = ((words[:, None] >> np.arange(n)) & 1).astype(np.uint8).reshape(-1)
    rx = np.packbits(bits, bitorder="little")
    assert_same(m, N, gpu_decode(m, rx, N), oracle.decode(m, rx, N))


# calls of at most this many coded bits take the small-call decoder (hamming.cu kSmallCallBits);
# larger ones the tile pipeline with the (7,4) / (15,11) / (31,26) table decoders
SMALL_CALL_BITS = 1 << 24


@pytest.mark.parametrize("m", [2, 3, 4])
def test_every_received_word_tiled_large(oracle, m):
    """Every received word of the code at N above the small-call limit (a
    ragged tail included), i.e. through the multi-CTA tile pipeline -- the
    (7,4) / (15,11) table decoders for m = 3, 4.  Each block of 2^n words is
    a fresh permutation, so every word lands on many codeword slots of a lane."""
    n = 2 ** m - 1
    rng = np.random.default_rng(1000 + m)
    N = max((1 << 17) + 77 if m < 4 else 4 * 2 ** n + 1234, SMALL_CALL_BITS // n + 77)
    blocks = (N + 2 ** n - 1) // 2 ** n
    words = np.concatenate([rng.permutation(2 ** n) for _ in range(blocks)]).astype(np.int64)[:N]
    bits = ((words[:, None] >> np.arange(n)) & 1).astype(np.uint8).reshape(-1)
    rx = np.packbits(bits, bitorder="little")
    assert_same(m, N, gpu_decode(m, rx, N), oracle.decode_mt(m, rx, N, THREADS))


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("N", [65535, 65536, 65537, 10 ** 6 + 13, "small_max", "small_max+1"])
def test_uniform_random_streams_large(oracle, m, N):
    """Uniformly random received bits (nearly every codeword erroneous, many
    with several flips) with garbage in the input pad bits: around 65 536
    codewords, at 10^6 + 13, and on both sides of the small-call limit (the
    largest call the small-call decoder takes, and one codeword more: the
    tile pipeline and, for m = 3..5, its table decoders)."""
    n = 2 ** m - 1
    if isinstance(N, str):
        N = SMALL_CALL_BITS // n + (1 if N.endswith("+1") else 0)
    rng = np.random.default_rng(m * 7919 + N)
    rx = rng.integers(0, 256, ham.coded_bytes(m, N), dtype=np.uint8)
    assert_same(m, N, gpu_decode(m, rx, N), oracle.decode_mt(m, rx, N, THREADS))


@pytest.mark.parametrize("m", [3, 5, 6])
def test_uniform_random_streams_and_pad_bits(oracle, m):
    """Uniformly random received bits (every codeword erroneous with high
    probability) and garbage in the input pad bits, which must be ignored."""
    rng = np.random.default_rng(m)
    for N in (1, 1000, 1024 + 5, 20_003):
        rx = rng.integers(0, 256, ham.coded_bytes(m, N), dtype=np.uint8)
        assert_same(m, N, gpu_decode(m, rx, N), oracle.decode(m, rx, N))


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_channel_corners(oracle, m):
    """p = 0 (nothing to correct), p = 1 single flips (paper regime: every
    error corrected), p = 1 with q2 = 1 (every codeword miscorrected)."""
    N = 3 * 1024 + 100
    for p, q2 in ((0.0, 0.0), (1.0, 0.0), (1.0, 1.0), (1e-3, 0.25)):
        rx, sent, err = oracle.generate(m, 77, 0, N, p=p, q2=q2, want_sent=True, want_err=True)
        got = gpu_decode(m, rx, N)
        want = oracle.decode(m, rx, N)
        assert_same(m, N, got, want)
        e = err.reshape(N, 2)
        if q2 == 0.0:
            assert np.array_equal(got[0], sent) and got[2] == int((e[:, 0] > 0).sum())
        if p == 1.0 and q2 == 1.0:
            assert got[2] == N


def test_empty_input_writes_zero_count():
    cnt = torch.full((1,), 12345, dtype=torch.int64, device="cuda")
    rx = torch.zeros(16, dtype=torch.uint8, device="cuda")
    data = torch.zeros(16, dtype=torch.uint8, device="cuda")
    ham.decode(6, rx, 0, data_out=data, syndromes=False, corrected=cnt)
    torch.cuda.synchronize()
    assert cnt.item() == 0


@pytest.mark.parametrize("m", [3, 6])
def test_canaries_past_the_end_untouched(oracle, m):
    N = 2 * 1024 + 77
    rx, _, _ = oracle.generate(m, 9, 0, N, p=0.3, q2=0.3)
    db, sb = ham.data_bytes(m, N), N
    data = torch.full((db + 64,), 0xA5, dtype=torch.uint8, device="cuda")
    syn = torch.full((sb + 64,), 0x5A, dtype=torch.uint8, device="cuda")
    rx_t = torch.full((rx.size + 64,), 0xFF, dtype=torch.uint8, device="cuda")
    rx_t[: rx.size] = gpu(rx)
    res = ham.decode(m, rx_t, N, data_out=data, syndromes=syn)
    torch.cuda.synchronize()
    d = data.cpu().numpy()
    s = syn.cpu().numpy()
    assert (d[db:] == 0xA5).all() and (s[sb:] == 0x5A).all()
    wd, ws, wc = oracle.decode(m, rx, N)
    assert np.array_equal(d[:db], wd) and np.array_equal(s[:sb], ws) and res.corrected.item() == wc


def test_repeated_calls_overwrite_count_and_are_deterministic(oracle):
    m, N = 5, 40_000
    rx, _, _ = oracle.generate(m, 3, 0, N, p=0.4, q2=0.2)
    a = gpu_decode(m, rx, N)
    b = gpu_decode(m, rx, N)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
def test_gpu_generator_matches_oracle_generator(oracle, m):
    """The GPU channel generator and the oracle's (written independently)
    produce byte-identical packets; any range regenerates on its own."""
    for c_first, N, p, q2 in ((0, 4681, 0.1, 0.0), (8 * 1000, 3 * 1024 + 9, 0.5, 0.5), (0, 2048, 1.0, 1.0),
                              (123456, 1500, 0.0, 0.0)):
        want, _, _ = oracle.generate(m, 0xBEEF, c_first, N, p=p, q2=q2)
        got = ham.channel_generate(m, 0xBEEF, c_first, N, p=p, q2=q2)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy()[: want.size], want), (m, c_first, N, p, q2)


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
def test_gpu_encoder_matches_oracle(oracle, m):
    n, k = oracle.code_nk(m)
    rng = np.random.default_rng(m)
    for N in (1, 100, 1024, 5000):
        data = rng.integers(0, 256, ham.data_bytes(m, N), dtype=np.uint8)
        want = oracle.encode(m, data, N)
        got = ham.encode(m, gpu(data), N)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy()[: want.size], want), (m, N)
        # round trip through the GPU decoder
        d, s, c = gpu_decode(m, got.cpu().numpy()[: want.size], N)
        full = np.unpackbits(data, bitorder="little")[: N * k]
        assert np.array_equal(np.unpackbits(d, bitorder="little")[: N * k], full) and c == 0


@pytest.mark.parametrize("m", [3, 6])
def test_decode_host_pipeline_matches_oracle(oracle, m):
    N = 9 * 1024 + 300
    rx, _, _ = oracle.generate(m, 21, 0, N, p=0.3, q2=0.3)
    want = oracle.decode(m, rx, N)
    chunk = 2048
    for streams in (1, 3):
        ws = torch.empty(ham.host_workspace_bytes(m, chunk, streams, True), dtype=torch.uint8, device="cuda")
        rx_h = torch.from_numpy(rx).pin_memory()
        data_h = torch.zeros(ham.data_bytes(m, N), dtype=torch.uint8).pin_memory()
        syn_h = torch.zeros(N, dtype=torch.uint8).pin_memory()
        cnt = ham.decode_host(m, rx_h, N, data_h, syn_h, ws, chunk_codewords=chunk, n_streams=streams)
        assert_same(m, N, (data_h.numpy(), syn_h.numpy(), cnt), want)


def _noisy_codewords(oracle, m, N, seed, p_flip=0.4):
    """Oracle-encoded random data with random single/double flips applied by
    numpy (channel simulation only)."""
    n, k = oracle.code_nk(m)
    rng = np.random.default_rng(seed)
    data = rng.integers(0, 256, (k * N + 7) // 8, dtype=np.uint8)
    rx = oracle.encode(m, data, N)
    bits = np.unpackbits(rx, bitorder="little")
    for c in np.nonzero(rng.random(N) < p_flip)[0]:
        for p in rng.choice(n, size=int(rng.integers(1, 3)), replace=False):
            bits[c * n + p] ^= 1
    return np.packbits(bits, bitorder="little")[: rx.size]


@pytest.mark.parametrize("m", [7, 8])
@pytest.mark.parametrize("N", [1, 31, 127, 128, 129, 255, 256, 257, 1000, 4097, 256 * 41, 300_001])
def test_long_perfect_codes_match_oracle(oracle, m, N):
    """(127,120) and (255,247) through the long-codeword engine."""
    rx = _noisy_codewords(oracle, m, N, 1000 * m + N)
    assert_same(m, N, gpu_decode(m, rx, N), oracle.decode(m, rx, N))


@pytest.mark.parametrize("m", [7, 8])
def test_long_perfect_codes_random_streams(oracle, m):
    rng = np.random.default_rng(m)
    for N in (5, 128 * 37 + 11):
        rx = rng.integers(0, 256, ham.coded_bytes(m, N), dtype=np.uint8)
        assert_same(m, N, gpu_decode(m, rx, N), oracle.decode(m, rx, N))


def _encoder_windows(N):
    """Codeword windows (start, count) checked against the oracle in the large
    encoder tests: starts are multiples of 8 so every window is byte-aligned
    in both the data and the coded stream; the last one ends at N."""
    last = (N - 4096) // 8 * 8
    return [(0, 4096), (N // 2 // 8 * 8, 4096), (last, N - last)]


@pytest.mark.parametrize("secded", [False, True])
@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_gpu_encoder_large_multi_round(oracle, m, secded):
    """~6M codewords: every warp of the persistent grid walks many tiles and
    wraps its TMA stage ring several times (the small encoder tests stay in the
    first round), plus a ragged tail.  Oracle-checked on three byte-aligned
    windows; the whole output round-trips through the (oracle-checked) GPU
    decoder with zero syndromes."""
    n, k = oracle.code_nk(m)
    w = (n + 1) if secded else n
    N = 6_000_003
    rng = np.random.default_rng(100 + m + 10 * secded)
    data = rng.integers(0, 256, ham.data_bytes(m, N), dtype=np.uint8)
    enc = ham.encode_secded if secded else ham.encode
    got = enc(m, gpu(data), N)
    torch.cuda.synchronize()
    out_bytes = (w * N + 7) // 8
    got_np = got.cpu().numpy()[:out_bytes]
    for c0, cnt in _encoder_windows(N):
        d0, d1 = c0 * k // 8, (c0 * k + cnt * k + 7) // 8
        want = (oracle.encode_secded if secded else oracle.encode)(m, np.ascontiguousarray(data[d0:d1]), cnt)
        o0 = c0 * w // 8
        assert np.array_equal(got_np[o0:o0 + want.size], want), (m, secded, c0)
    if secded:
        res = ham.decode_secded(m, got, N)
        torch.cuda.synchronize()
        assert int(res.counts.cpu().numpy().sum()) == 0
    else:
        res = ham.decode(m, got, N)
        torch.cuda.synchronize()
        assert int(res.corrected.item()) == 0
    dec = res.data.cpu().numpy()[: ham.data_bytes(m, N)]
    assert np.array_equal(np.unpackbits(dec, bitorder="little")[: N * k],
                          np.unpackbits(data, bitorder="little")[: N * k])


@pytest.mark.parametrize("m,N0", [(3, 4681), (4, 2000), (6, 2000), (4, 500_000), (6, 200_000)])
def test_chained_small_calls_keep_stream_order(oracle, m, N0):
    """Small calls launch with programmatic dependent launch: a call whose INPUT is the
    previous call's OUTPUT (decode -> decode of the data stream as a new received stream, five deep,
    eagerly and inside one CUDA graph) must still see the finished output, and each count stays its own."""
    n, k = ham.code_nk(m)
    # N0 > one CTA's share (14336 / 3072 codewords for m = 4 / 6): multi-CTA small calls, whose count
    # goes through the stream's launch slot eagerly and through a memset + atomics under capture
    rx_np, _, _ = oracle.generate(m, 0xC4A1 + m, 0, N0, p=0.3, q2=0.2)
    # oracle chain: level i decodes the previous level's data bytes as a packet of N_i codewords
    want, cur, N = [], rx_np, N0
    for _ in range(5):
        wd, ws, wc = oracle.decode(m, cur, N)
        want.append((N, wd, ws, wc))
        N = wd.size * 8 // n
        cur = wd
    for mode in ("eager", "graph"):
        bufs, N = [], N0
        src = gpu(rx_np)
        for (Ni, wd, _, _) in want:
            bufs.append((src, Ni, torch.empty(ham.data_bytes(m, Ni), dtype=torch.uint8, device="cuda"),
                         torch.empty(Ni, dtype=torch.uint8, device="cuda"), torch.empty(1, dtype=torch.int64, device="cuda")))
            src = bufs[-1][2]
        def run():
            for s, Ni, d, sy, c in bufs:
                ham.decode(m, s, Ni, data_out=d, syndromes=sy, corrected=c)
        if mode == "eager":
            run()
        else:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                run()  # warm (tables, launch slots) outside capture
                for _, _, d, sy, c in bufs:
                    d.zero_(), sy.zero_(), c.zero_()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    run()
            torch.cuda.synchronize()
            for _, _, d, sy, c in bufs:
                d.zero_(), sy.zero_(), c.fill_(-1)
            g.replay()
        torch.cuda.synchronize()
        for (Ni, wd, ws, wc), (_, _, d, sy, c) in zip(want, bufs):
            assert np.array_equal(d.cpu().numpy()[: wd.size], wd), (mode, m, Ni)
            assert np.array_equal(sy.cpu().numpy(), ws), (mode, m, Ni)
            assert int(c.item()) == wc, (mode, m, Ni)
