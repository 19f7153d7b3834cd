"""Pins for the oracle's seeded channel generator."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vectors(oracle):
    """Seed 0, codeword 0: the message is the low k bits of the first
    splitmix64 output from state 0 (public reference vector)."""
    with open(os.path.join(GOLDEN, "splitmix64_vectors.json")) as f:
        g = json.load(f)
    u0 = int(g["outputs"][0], 16)
    for m in (2, 3, 4, 5, 6):
        n, k = oracle.code_nk(m)
        _, sent, err = oracle.generate(m, 0, 0, 1, p=0.0, want_sent=True, want_err=True)
        got = int.from_bytes(sent.tobytes(), "little")
        assert got == u0 & ((1 << k) - 1)
        assert err.tolist() == [0, 0]
    # u(0,1) = second output decides the event: with p just above/below it
    u1 = int(g["outputs"][1], 16)
    _, _, err = oracle.generate(6, 0, 0, 1, p=(u1 + 2 ** 40) / 2 ** 64, want_err=True)
    assert err[0] != 0
    _, _, err = oracle.generate(6, 0, 0, 1, p=(u1 - 2 ** 40) / 2 ** 64, want_err=True)
    assert err[0] == 0


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
def test_generator_determinism_and_ranges(oracle, m):
    n, k = oracle.code_nk(m)
    a = oracle.generate(m, 1234, 0, 4000, p=0.3, q2=0.5, want_sent=True, want_err=True)
    b = oracle.generate(m, 1234, 0, 4000, p=0.3, q2=0.5, want_sent=True, want_err=True, threads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    c = oracle.generate(m, 1235, 0, 4000, p=0.3, q2=0.5)
    assert not np.array_equal(a[0], c[0])
    # any range regenerates on its own (draws depend on the global index only)
    sub = oracle.generate(m, 1234, 800, 1600, p=0.3, q2=0.5, want_sent=True, want_err=True)
    full_bits = np.unpackbits(a[0], bitorder="little")
    sub_bits = np.unpackbits(sub[0], bitorder="little")
    assert np.array_equal(full_bits[800 * n: 2400 * n], sub_bits[: 1600 * n])
    assert np.array_equal(a[2][1600:4800], sub[2])


@pytest.mark.parametrize("m", [3, 6])
def test_generator_error_model(oracle, m):
    n, k = oracle.code_nk(m)
    N = 20000
    rx, sent, err = oracle.generate(m, 99, 0, N, p=0.0, want_sent=True, want_err=True)
    assert not err.any()
    data, syn, cnt = oracle.decode(m, rx, N)
    assert np.array_equal(data, sent) and cnt == 0
    # p = 1, q2 = 0: exactly one flip per codeword, all corrected
    rx, sent, err = oracle.generate(m, 99, 0, N, p=1.0, q2=0.0, want_sent=True, want_err=True)
    e = err.reshape(N, 2)
    assert (e[:, 0] >= 1).all() and (e[:, 0] <= n).all() and not e[:, 1].any()
    data, syn, cnt = oracle.decode(m, rx, N)
    assert np.array_equal(data, sent) and cnt == N
    assert np.array_equal(syn, e[:, 0])
    # p = 1, q2 = 1: two distinct flips everywhere; s = p1 ^ p2
    rx, sent, err = oracle.generate(m, 99, 0, N, p=1.0, q2=1.0, want_err=True)
    e = err.reshape(N, 2).astype(int)
    assert (e[:, 0] != e[:, 1]).all() and (e[:, 1] >= 1).all() and (e[:, 1] <= n).all()
    _, syn, cnt = oracle.decode(m, rx, N)
    assert np.array_equal(syn, (e[:, 0] ^ e[:, 1]).astype(np.uint8)) and cnt == N
    # event rate ~ p, weight-2 share ~ q2 (binomial 5-sigma bounds)
    p, q2 = 0.1, 0.25
    _, _, err = oracle.generate(m, 5, 0, N, p=p, q2=q2, want_err=True)
    e = err.reshape(N, 2)
    ev = int((e[:, 0] > 0).sum())
    assert abs(ev - N * p) < 5 * np.sqrt(N * p * (1 - p))
    w2 = int((e[:, 1] > 0).sum())
    assert abs(w2 - ev * q2) < 5 * np.sqrt(ev * q2 * (1 - q2))
    # positions are roughly uniform over [1, n]
    hist = np.bincount(e[e[:, 0] > 0, 0], minlength=n + 1)[1:]
    assert hist.min() > 0


def test_threaded_decode_matches_single(oracle):
    for m in (3, 4, 5, 6):
        rx, _, _ = oracle.generate(m, 3, 0, 12345, p=0.5, q2=0.3)
        a = oracle.decode(m, rx, 12345)
        b = oracle.decode_mt(m, rx, 12345, threads=5)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
