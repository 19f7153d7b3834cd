"""GPU parity (-m gpu) for extended Hamming / SECDED:
decode, encode and the channel generator against the CPU oracle, bit for bit,
including double errors (detected, never miscorrected) and every received
word of the (8,4) and (16,11) codes."""
import numpy as np
import pytest
import torch

import paper_1412_6862_b200 as ham

pytestmark = pytest.mark.gpu

SIZES = [1, 33, 1023, 1024, 1025, 3 * 1024 + 77, 70_000]


def gpu_decode(m, rx_np, N, flags=True):
    res = ham.decode_secded(m, torch.from_numpy(rx_np).cuda(), N, flags=flags)
    torch.cuda.synchronize()
    return (res.data.cpu().numpy()[: ham.data_bytes(m, N)],
            None if res.flags is None else res.flags.cpu().numpy()[:N], res.counts.cpu().tolist())


@pytest.mark.parametrize("m", [3, 4, 5, 6])
@pytest.mark.parametrize("N", SIZES)
def test_decode_secded_matches_oracle(oracle, m, N):
    rx, _, _ = oracle.generate_secded(m, 0x5EC + N, 0, N, p=0.6, q2=0.4)
    wd, wf, c1, c2 = oracle.decode_secded(m, rx, N)
    d, f, c = gpu_decode(m, rx, N)
    assert np.array_equal(d, wd) and np.array_equal(f, wf) and c == [c1, c2]
    d2, f2, c2b = gpu_decode(m, rx, N, flags=False)
    assert f2 is None and np.array_equal(d2, wd) and c2b == [c1, c2]


@pytest.mark.parametrize("m", [3, 4])
def test_every_received_word(oracle, m):
    w = 2 ** m
    N = 2 ** w
    words = np.arange(N, dtype=np.int64)
    rx = np.packbits(((words[:, None] >> np.arange(w)) & 1).astype(np.uint8).reshape(-1), bitorder="little")
    wd, wf, c1, c2 = oracle.decode_secded(m, rx, N)
    d, f, c = gpu_decode(m, rx, N)
    assert np.array_equal(d, wd) and np.array_equal(f, wf) and c == [c1, c2]


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_generator_and_encoder_match_oracle(oracle, m):
    for c_first, N, p, q2 in ((0, 4681, 0.1, 0.0), (8000, 3 * 1024 + 9, 1.0, 0.5), (0, 2048, 1.0, 1.0)):
        want, sent, _ = oracle.generate_secded(m, 0xFEED, c_first, N, p=p, q2=q2, want_sent=True)
        got = ham.channel_generate_secded(m, 0xFEED, c_first, N, p=p, q2=q2)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy()[: want.size], want), (m, c_first, N)
        enc = ham.encode_secded(m, torch.from_numpy(sent).cuda(), N)
        torch.cuda.synchronize()
        assert np.array_equal(enc.cpu().numpy()[: want.size], oracle.encode_secded(m, sent, N))


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_secded_large_counts(oracle, m):
    """A 1 GiB SECDED stream (the multi-CTA table / POPC decoders): corrected +
    detected counts equal the channel's single / double events (closed form),
    flags agree with counts, a window matches the oracle."""
    N = (1 << 30) * 8 // (1 << m)
    rx = ham.channel_generate_secded(m, 99, 0, N, p=0.2, q2=0.3)
    res = ham.decode_secded(m, rx, N)
    torch.cuda.synchronize()
    c1, c2 = res.counts.cpu().tolist()
    f = res.flags[:N]
    assert c1 == int((f & 0x40 != 0).sum().item()) and c2 == int((f & 0x80 != 0).sum().item())
    assert abs(c1 - N * 0.2 * 0.7) < 6 * np.sqrt(N * 0.2 * 0.7) and abs(c2 - N * 0.2 * 0.3) < 6 * np.sqrt(N * 0.06)
    # a window against the oracle, regenerated on its own
    c0, w = (N // 2) // 8 * 8, 1 << 14
    rxw, _, _ = oracle.generate_secded(m, 99, c0, w, p=0.2, q2=0.3)
    wd, wf, _, _ = oracle.decode_secded(m, rxw, w)
    k = 2 ** m - 1 - m
    assert np.array_equal(res.data[c0 * k // 8: c0 * k // 8 + wd.size - 1].cpu().numpy(), wd[:-1])
    assert np.array_equal(f[c0: c0 + w].cpu().numpy(), wf)


@pytest.mark.parametrize("m", [3, 4, 5, 6])
@pytest.mark.parametrize("N", [65535, 65536, 65537, 10 ** 6 + 13])
def test_uniform_random_streams_large(oracle, m, N):
    """Uniformly random SECDED words (single, double and heavier errors in
    every mix) through the multi-CTA table / POPC decoders (>= 65 536
    codewords) and the small launch just below."""
    rng = np.random.default_rng(m * 131 + N)
    rx = rng.integers(0, 256, ham.secded_coded_bytes(m, N), dtype=np.uint8)
    wd, wf, c1, c2 = oracle.decode_secded(m, rx, N)
    d, f, c = gpu_decode(m, rx, N)
    assert np.array_equal(d, wd) and np.array_equal(f, wf) and c == [c1, c2]
