"""Pins for the oracle's extended-Hamming (SECDED) routines (SURVEY.md 8(f) f4,
DESIGN.md reading R17) against the textbook characterisation of the extended
code: minimum distance 4; every single error (including in the parity bit)
corrected; every double error detected and never miscorrected -- checked by
brute force over all received words for m = 3, 4."""
import itertools

import numpy as np
import pytest


def popcount(v):
    return bin(int(v)).count("1")


@pytest.mark.parametrize("m", [3, 4])
def test_secded_bruteforce(oracle, m):
    n = 2 ** m - 1
    k = n - m
    w = n + 1
    N = 2 ** k
    data = np.packbits(((np.arange(N)[:, None] >> np.arange(k)) & 1).astype(np.uint8).reshape(-1), bitorder="little")
    rx = oracle.encode_secded(m, data, N)
    bits = np.unpackbits(rx, bitorder="little").reshape(N, w)
    cw = (bits.astype(np.int64) << np.arange(w)).sum(1)
    # the extended code: even weight, minimum distance 4, positions 1..n a Hamming codeword
    assert all(popcount(v) % 2 == 0 for v in cw)
    d = np.bitwise_count(cw[:, None] ^ cw[None, :])
    assert d[~np.eye(N, dtype=bool)].min() == 4
    # every received word of length w
    words = np.arange(2 ** w, dtype=np.int64)
    stream = np.packbits(((words[:, None] >> np.arange(w)) & 1).astype(np.uint8).reshape(-1), bitorder="little")
    out, flags, c1, c2 = oracle.decode_secded(m, stream, 2 ** w)
    got = np.unpackbits(out, bitorder="little")[: (2 ** w) * k].reshape(-1, k)
    got_int = (got.astype(np.int64) << np.arange(k)).sum(1)
    dist = np.bitwise_count(words[:, None] ^ cw[None, :])
    dmin = dist.min(1)
    near = dist.argmin(1)
    one = dmin <= 1
    assert np.array_equal(got_int[one], near[one])                       # corrected (or clean)
    assert ((flags[dmin == 1] & 0x40) != 0).all() and not (flags[dmin == 0] & 0xC0).any()
    two = dmin == 2
    assert ((flags[two] & 0x80) != 0).all() and not (flags[two] & 0x40).any()   # detected, not corrected
    assert c1 == int((dmin == 1).sum()) and c2 == int(two.sum())
    # the syndrome field is the XOR of the set positions 1..n
    s = np.zeros(2 ** w, np.int64)
    for p in range(1, w):
        s ^= np.where((words >> p) & 1, p, 0)
    assert np.array_equal(flags & 0x3F, s)


@pytest.mark.parametrize("m", [3, 4, 5, 6])
def test_secded_generator_and_roundtrip(oracle, m):
    n = 2 ** m - 1
    N = 5000
    rx, sent, err = oracle.generate_secded(m, 3, 0, N, p=1.0, q2=0.5, want_sent=True, want_err=True)
    e = err.reshape(N, 2).astype(int)
    assert (e[:, 0] >= 1).all() and (e[:, 0] <= n + 1).all()
    two = e[:, 1] > 0
    assert (e[two, 0] != e[two, 1]).all()
    data, flags, c1, c2 = oracle.decode_secded(m, rx, N)
    assert c1 == int((~two).sum()) and c2 == int(two.sum())
    k = n - m
    got = np.unpackbits(data, bitorder="little")[: N * k].reshape(N, k)
    want = np.unpackbits(sent, bitorder="little")[: N * k].reshape(N, k)
    assert np.array_equal(got[~two], want[~two])        # every single error corrected
    rx0, sent0, _ = oracle.generate_secded(m, 3, 0, N, p=0.0, want_sent=True)
    data0, flags0, a, b = oracle.decode_secded(m, rx0, N)
    assert np.array_equal(data0, sent0) and a == b == 0 and not flags0.any()
    assert np.array_equal(oracle.encode_secded(m, sent0, N), rx0)
