"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: the
paper's printed worked example, SPEC.md's examples, textbook
closed forms of the Hamming code, brute-force nearest-codeword decoding over
every received word for m <= 4, and hand-derived byte layouts.  A plausible
mistake in oracle/oracle.c (dropped index-set member, wrong syndrome bit
weight, flipped bit order, parity at the wrong position, off-by-one in the
correction) fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def bits(s):
    return np.array([int(ch) for ch in s], np.uint8)


def positions_xor(word_bits):
    """Textbook closed form (independent of index sets): the syndrome of a
    Hamming word is the XOR of the 1-based positions of its set bits."""
    s = 0
    for p, b in enumerate(word_bits, start=1):
        if b:
            s ^= p
    return s


def is_pow2(p):
    return p & (p - 1) == 0


# ------------------------------------------------------------------ paper
def test_paper_index_sets_n11(oracle):
    g = load("paper_index_sets.json")
    assert oracle.lib().oracle_parity_positions(g["n"]) == g["r"]
    for j, expect in enumerate(g["index_sets"]):
        assert oracle.index_set(j, g["n"]) == expect
    with pytest.raises(ValueError):
        oracle.index_set(g["r"], g["n"])        # only r sets exist (reading R6)


def test_paper_parity_count_n11(oracle):
    # |H_i| = 7 + 4 = 11 and |R| = 4  -> k = 7 needs r = 4.
    assert oracle.parity_bit_count(7) == 4


# ------------------------------------------------------------------- spec
def test_spec_examples(oracle):
    g = load("spec_examples.json")
    for e in g["parity_bit_count"]:
        assert oracle.parity_bit_count(e["k"]) == e["r"], e["cite"]
    for e in g["index_set"]:
        assert oracle.index_set(e["j"], e["n"]) == e["set"], e["cite"]
    for e in g["encode"]:
        assert "".join(map(str, oracle.encode_bits(e["n"], bits(e["message"])))) == e["codeword"], e["cite"]
    for e in g["syndrome"]:
        assert oracle.syndrome_bits(e["n"], bits(e["received"])) == e["s"], e["cite"]
    for e in g["detect_and_correct"]:
        out, st = oracle.correct_bits(e["n"], bits(e["received"]), e["s"])
        assert st == e["status"], e["cite"]
        assert "".join(map(str, out)) == e["corrected"], e["cite"]
    for e in g["remove_redundancy"]:
        got = oracle.remove_redundancy_bits(e["n"], bits(e["codeword"]))
        assert "".join(map(str, got)) == e["message"], e["cite"]
    for e in g["checksum_kernel"]:
        rng = np.random.default_rng(11)
        for _ in range(20):
            cw = oracle.encode_bits(e["n"], rng.integers(0, 2, 7, dtype=np.uint8))
            cw[e["flip"] - 1] ^= 1
            assert oracle.syndrome_bits(e["n"], cw) == e["s"], e["cite"]


def test_parity_bit_count_monotone_and_minimal(oracle):
    prev = 0
    for k in range(1, 3000):
        r = oracle.parity_bit_count(k)
        assert r >= prev
        assert 2 ** r >= k + r + 1 and 2 ** (r - 1) < k + (r - 1) + 1
        prev = r
    assert oracle.parity_bit_count(0) == -1


def test_index_set_contains_parity_position(oracle):
    for n in (3, 7, 11, 15, 31, 63, 100, 1611):
        r = oracle.lib().oracle_parity_positions(n)
        for j in range(r):
            s = oracle.index_set(j, n)
            assert (1 << j) in s and max(s) <= n and s == sorted(s)
            assert all((p >> j) & 1 for p in s)
            assert len(s) == sum(1 for p in range(1, n + 1) if (p >> j) & 1)


# --------------------------------------------------- textbook closed forms
@pytest.mark.parametrize("n", [3, 7, 11, 15, 31, 63, 100, 127, 255])
def test_syndrome_is_xor_of_set_positions(oracle, n):
    rng = np.random.default_rng(n)
    words = [rng.integers(0, 2, n, dtype=np.uint8) for _ in range(300)]
    if n <= 11:
        words += [np.array(w, np.uint8) for w in itertools.product((0, 1), repeat=n)]
    for w in words:
        assert oracle.syndrome_bits(n, w) == positions_xor(w)


@pytest.mark.parametrize("n", [3, 7, 11, 15, 31, 63, 1611])
def test_encoder_places_message_and_zeroes_syndrome(oracle, n):
    r = oracle.lib().oracle_parity_positions(n)
    k = n - r
    rng = np.random.default_rng(n + 1)
    data_pos = [p for p in range(1, n + 1) if not is_pow2(p)]
    assert len(data_pos) == k
    for _ in range(200):
        msg = rng.integers(0, 2, k, dtype=np.uint8)
        cw = oracle.encode_bits(n, msg)
        assert positions_xor(cw) == 0                 # H x = 0 (textbook)
        assert np.array_equal(cw[np.array(data_pos) - 1], msg)   # reading R3
        assert np.array_equal(oracle.remove_redundancy_bits(n, cw), msg)


@pytest.mark.parametrize("m", [2, 3, 4])
def test_codebook_is_the_perfect_hamming_code(oracle, m):
    """Exhaustive: 2^k distinct codewords, linear, minimum distance 3,
    exactly the words with XOR-of-positions 0, and radius-1 spheres tile
    {0,1}^n (2^k (n+1) = 2^n)."""
    n = 2 ** m - 1
    k = n - m
    cws = np.array([oracle.encode_bits(n, np.array(msg, np.uint8))
                    for msg in itertools.product((0, 1), repeat=k)], np.uint8)
    ints = cws.astype(np.int64) @ (1 << np.arange(n, dtype=np.int64))
    assert len(set(ints.tolist())) == 2 ** k
    # the same set as {x : XOR of positions of set bits = 0}
    all_words = np.arange(2 ** n, dtype=np.int64)
    synd = np.zeros_like(all_words)
    for p in range(1, n + 1):
        synd ^= np.where((all_words >> (p - 1)) & 1, p, 0)
    assert set(all_words[synd == 0].tolist()) == set(ints.tolist())
    # linearity and minimum distance
    s = set(ints.tolist())
    a = ints[:, None] ^ ints[None, :]
    assert all(v in s for v in np.unique(a).tolist())
    w = np.array([bin(v).count("1") for v in np.unique(a).tolist() if v])
    assert w.min() == 3
    assert 2 ** k * (n + 1) == 2 ** n


@pytest.mark.parametrize("m", [2, 3, 4])
def test_decode_equals_bruteforce_nearest_codeword(oracle, m):
    """Every received word r of length n: the oracle's data output equals the
    message of the (unique) codeword at Hamming distance <= 1 found by brute
    force over the whole codebook, and the syndrome is the position where they
    differ (0 if none)."""
    n = 2 ** m - 1
    k = n - m
    msgs = list(itertools.product((0, 1), repeat=k))
    cw_int = np.array([int("".join(map(str, oracle.encode_bits(n, np.array(mm, np.uint8))[::-1])), 2)
                       for mm in msgs], np.int64)
    msg_int = np.array([sum(b << i for i, b in enumerate(mm)) for mm in msgs], np.int64)
    # pack every received word into one stream and decode it in one call
    N = 2 ** n
    words = np.arange(N, dtype=np.int64)
    stream_bits = ((words[:, None] >> np.arange(n)) & 1).astype(np.uint8).reshape(-1)
    rx = np.packbits(stream_bits, bitorder="little")
    data, syn, cnt = oracle.decode(m, rx, N)
    out_bits = np.unpackbits(data, bitorder="little")[: N * k].reshape(N, k)
    out_int = (out_bits.astype(np.int64) << np.arange(k)).sum(1)
    for r0 in range(0, N, 4096):
        r = words[r0:r0 + 4096]
        d = np.bitwise_count(r[:, None] ^ cw_int[None, :]).astype(np.int64)
        best = d.argmin(1)
        assert (d.min(1) <= 1).all()                         # perfect code
        assert ((d <= 1).sum(1) == 1).all()                  # unique within radius 1
        assert np.array_equal(out_int[r0:r0 + 4096], msg_int[best])
        diff = r ^ cw_int[best]
        pos = np.where(diff == 0, 0, np.log2(np.maximum(diff, 1)).astype(np.int64) + 1)
        assert np.array_equal(syn[r0:r0 + 4096].astype(np.int64), pos)
    assert cnt == N - 2 ** k


@pytest.mark.parametrize("m", [3, 4])
def test_exhaustive_single_error_correction(oracle, m):
    """North star: every data word with every single-bit error position is
    corrected, and the syndrome equals the error position (m = 3, 4)."""
    n = 2 ** m - 1
    k = n - m
    msgs = np.array(list(itertools.product((0, 1), repeat=k)), np.uint8)
    cws = np.array([oracle.encode_bits(n, mm) for mm in msgs])
    rows, want_syn, want_msg = [], [], []
    for i in range(len(msgs)):
        for p in range(1, n + 1):
            r = cws[i].copy()
            r[p - 1] ^= 1
            rows.append(r)
            want_syn.append(p)
            want_msg.append(msgs[i])
    rx = np.packbits(np.concatenate(rows), bitorder="little")
    N = len(rows)
    data, syn, cnt = oracle.decode(m, rx, N)
    got = np.unpackbits(data, bitorder="little")[: N * k].reshape(N, k)
    assert np.array_equal(got, np.array(want_msg))
    assert np.array_equal(syn, np.array(want_syn, np.uint8))
    assert cnt == N


@pytest.mark.parametrize("m", [5, 6])
def test_single_error_every_position_random_words(oracle, m):
    n = 2 ** m - 1
    k = n - m
    rng = np.random.default_rng(m)
    msgs = rng.integers(0, 2, (300, k), dtype=np.uint8)
    rows, want_syn, want_msg = [], [], []
    for mm in msgs:
        cw = oracle.encode_bits(n, mm)
        for p in range(1, n + 1):
            r = cw.copy()
            r[p - 1] ^= 1
            rows.append(r)
            want_syn.append(p)
            want_msg.append(mm)
    N = len(rows)
    data, syn, cnt = oracle.decode(m, np.packbits(np.concatenate(rows), bitorder="little"), N)
    got = np.unpackbits(data, bitorder="little")[: N * k].reshape(N, k)
    assert np.array_equal(got, np.array(want_msg))
    assert np.array_equal(syn, np.array(want_syn, np.uint8))
    assert cnt == N


@pytest.mark.parametrize("m", [3, 4])
def test_double_error_miscorrects_to_distance_three(oracle, m):
    """Reading R9: two flips p1 != p2 give s = p1 xor p2 (nonzero), and the
    decoder lands on a codeword at distance exactly 3 from the one sent."""
    n = 2 ** m - 1
    k = n - m
    rng = np.random.default_rng(7 + m)
    rows, sent, pairs = [], [], []
    for _ in range(40):
        mm = rng.integers(0, 2, k, dtype=np.uint8)
        cw = oracle.encode_bits(n, mm)
        for p1 in range(1, n + 1):
            for p2 in range(p1 + 1, n + 1):
                r = cw.copy()
                r[p1 - 1] ^= 1
                r[p2 - 1] ^= 1
                rows.append(r)
                sent.append(cw)
                pairs.append((p1, p2))
    N = len(rows)
    data, syn, cnt = oracle.decode(m, np.packbits(np.concatenate(rows), bitorder="little"), N)
    got = np.unpackbits(data, bitorder="little")[: N * k].reshape(N, k)
    assert np.array_equal(syn, np.array([a ^ b for a, b in pairs], np.uint8))
    assert cnt == N
    for i in range(0, N, 97):
        dec_cw = oracle.encode_bits(n, got[i])
        assert int((dec_cw != sent[i]).sum()) == 3


# ------------------------------------------------------- stream layout pins
def test_stream_byte_layout_pins(oracle):
    g = load("stream_layout_pins.json")
    for c in g["cases"]:
        if c["what"] == "encode":
            rx = oracle.encode(c["m"], np.array(c["data"], np.uint8), c["count"])
            assert rx.tolist() == c["rx"], c
        else:
            data, syn, cnt = oracle.decode(c["m"], np.array(c["rx"], np.uint8), c["count"])
            assert data.tolist() == c["data"], c
            assert syn.tolist() == c["syn"], c
            assert cnt == c["corrected"], c


def test_msb_first_layout_would_fail_pin(oracle):
    # The 0x76 pin discriminates bit order: MSB-first packing gives 0x6E.
    cw = bits("0110111")
    assert int(np.packbits(np.append(cw, 0), bitorder="big")[0]) == 0x6E
    assert int(np.packbits(np.append(cw, 0), bitorder="little")[0]) == 0x76


@pytest.mark.parametrize("m", [2, 3, 4, 5, 6])
@pytest.mark.parametrize("count", [1, 7, 8, 9, 33, 1000])
def test_stream_roundtrip_and_padding(oracle, m, count):
    n, k = oracle.code_nk(m)
    rng = np.random.default_rng(count * 10 + m)
    data = np.packbits(rng.integers(0, 2, k * count, dtype=np.uint8), bitorder="little")
    rx = oracle.encode(m, data, count)
    assert rx.size == (n * count + 7) // 8
    if (n * count) % 8:
        assert rx[-1] >> ((n * count) % 8) == 0
    out, syn, cnt = oracle.decode(m, rx, count)
    assert np.array_equal(out, data) and cnt == 0 and not syn.any()
    # pad bits of the input are ignored; pad bits of the output are written 0
    rx2 = rx.copy()
    if (n * count) % 8:
        rx2[-1] |= np.uint8((0xFF << ((n * count) % 8)) & 0xFF)
    out2, _, _ = oracle.decode(m, rx2, count)
    assert np.array_equal(out2, data)
