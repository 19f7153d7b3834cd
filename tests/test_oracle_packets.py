"""Pins for the oracle's packet routines -- the paper's own workload (a packet
of M message bytes split into t shortened-Hamming segments),
SURVEY.md 8(f) row f2."""
import itertools
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def positions_xor(bits):
    s = 0
    for p, b in enumerate(bits, start=1):
        if b:
            s ^= p
    return s


def test_spec_make_layout(oracle):
    with open(os.path.join(GOLDEN, "spec_packet_examples.json")) as f:
        g = json.load(f)
    for e in g["make_layout"]:
        k, n, total = oracle.packet_layout(e["bits"], e["t"])
        assert k == e["seg_k"], e["cite"]
        if "seg_n" in e:
            assert n == e["seg_n"], e["cite"]
        assert total == sum(n)


@pytest.mark.parametrize("M", [400, 800, 1200, 1600, 2000, 1, 7, 1024])
@pytest.mark.parametrize("t", [1, 2, 3, 4, 5, 6, 7])
def test_layout_invariants(oracle, M, t):
    bits = 8 * M
    if bits < t:
        return
    k, n, total = oracle.packet_layout(bits, t)
    assert sum(k) == bits and max(k) - min(k) <= 1 and k == sorted(k, reverse=True)
    for kk, nn in zip(k, n):
        r = nn - kk
        assert 2 ** r >= kk + r + 1 and 2 ** (r - 1) < kk + r   # minimal r
    if (M, t) == (2000, 2):
        assert n == [8013, 8013]                                 # the paper grid tops out at n = 8013
    if (M, t) == (400, 6):
        assert max(n) == 544


@pytest.mark.parametrize("k", range(1, 11))
def test_exhaustive_single_error_shortened_codes(oracle, k):
    """SPEC acceptance #2: every k in 1..10, every message, every single flip."""
    r = oracle.parity_bit_count(k)
    n = k + r
    for msg in itertools.product((0, 1), repeat=k):
        msg = np.array(msg, np.uint8)
        cw = oracle.encode_bits(n, msg)
        assert positions_xor(cw) == 0
        for p in range(1, n + 1):
            rx = cw.copy()
            rx[p - 1] ^= 1
            s = oracle.syndrome_bits(n, rx)
            assert s == p
            fixed, st = oracle.correct_bits(n, rx, s)
            assert st == 1 and np.array_equal(oracle.remove_redundancy_bits(n, fixed), msg)


def test_bruteforce_shortened_n11(oracle):
    """All 2^11 received words of the paper's n = 11 code: a word within
    distance 1 of a codeword decodes to it; every other word has s != 0 and is
    either flagged (s > 11) or lands on the codeword that flipping s gives."""
    n, k = 11, 7
    book = {}
    for msg in itertools.product((0, 1), repeat=k):
        cw = oracle.encode_bits(n, np.array(msg, np.uint8))
        book[tuple(cw.tolist())] = np.array(msg, np.uint8)
    assert len(book) == 2 ** k
    cws = np.array(list(book.keys()), np.uint8)
    for w in itertools.product((0, 1), repeat=n):
        w = np.array(w, np.uint8)
        d = (cws != w).sum(1)
        s = oracle.syndrome_bits(n, w)
        assert s == positions_xor(w)
        if d.min() <= 1:
            best = cws[d.argmin()]
            fixed, st = oracle.correct_bits(n, w, s)
            assert np.array_equal(fixed, best)
        else:
            assert s != 0
            fixed, st = oracle.correct_bits(n, w, s)
            if s > n:
                assert st == -1
            else:
                assert st == 1 and tuple(fixed.tolist()) in book


@pytest.mark.parametrize("M,t", [(400, 2), (400, 6), (800, 3), (1200, 4), (1600, 5), (2000, 2), (2000, 6), (13, 3)])
def test_packet_roundtrip_and_one_error_per_segment(oracle, M, t):
    rng = np.random.default_rng(M * 10 + t)
    k, n, total = oracle.packet_layout(8 * M, t)
    for _ in range(3):
        msg = rng.integers(0, 256, M, dtype=np.uint8)
        rx = oracle.encode_packet(M, t, msg)
        assert rx.size == (total + 7) // 8
        out, syn, st = oracle.decode_packet(M, t, rx)
        assert np.array_equal(out, msg) and st == 0 and not syn.any()
        # the paper's regime: one error in every segment (t errors per packet)
        bits = np.unpackbits(rx, bitorder="little")
        off = 0
        pos = []
        for nn in n:
            p = int(rng.integers(1, nn + 1))
            bits[off + p - 1] ^= 1
            pos.append(p)
            off += nn
        out, syn, st = oracle.decode_packet(M, t, np.packbits(bits, bitorder="little"))
        assert np.array_equal(out, msg) and st == 1 and syn.tolist() == pos


def test_uncorrectable_segment(oracle):
    with open(os.path.join(GOLDEN, "spec_packet_examples.json")) as f:
        g = json.load(f)["uncorrectable"]
    # one segment of 7 message bits is the n = 11 code
    msg = np.array([0x5A], np.uint8)
    M, t = 1, 1
    k, n, _ = oracle.packet_layout(8, 1)
    assert n == [12]   # 8 message bits need r = 4: n = 12 (positions 1..12)
    rx = oracle.encode_packet(M, t, msg)
    bits = np.unpackbits(rx, bitorder="little")
    for p in g["flips"]:
        bits[p - 1] ^= 1
    out, syn, st = oracle.decode_packet(M, t, np.packbits(bits, bitorder="little"))
    assert int(syn[0]) == g["s"] and st == 1   # 12 <= n = 12 here: a (mis)correction, not a failure
    # with n = 11 (7 message bits) the same syndrome names no position: uncorrectable
    cw = oracle.encode_bits(11, np.array([1, 0, 1, 1, 0, 1, 0], np.uint8))
    for p in g["flips"]:
        cw[p - 1] ^= 1
    assert oracle.syndrome_bits(11, cw) == 12
    assert oracle.correct_bits(11, cw, 12)[1] == -1


def test_packet_generator(oracle):
    M, t = 400, 3
    stride = (oracle.packet_coded_bytes(M, t) + 15) // 16 * 16
    a, msg = oracle.generate_packets(M, t, 7, 0, 20, stride, p=1.0, want_msg=True)
    b, _ = oracle.generate_packets(M, t, 7, 0, 20, stride, p=1.0, want_msg=True, threads=3)
    assert np.array_equal(a, b)
    c, _ = oracle.generate_packets(M, t, 7, 5, 10, stride, p=1.0)
    assert np.array_equal(a[5 * stride: 15 * stride], c)
    out, syn, st = oracle.decode_packets(M, t, a, 20, stride, threads=2)
    assert np.array_equal(out, msg) and (st == 1).all() and (syn > 0).all()
    z, msg0 = oracle.generate_packets(M, t, 7, 0, 20, stride, p=0.0, want_msg=True)
    out, syn, st = oracle.decode_packets(M, t, z, 20, stride)
    assert np.array_equal(out, msg0) and (st == 0).all() and not syn.any()
    assert np.array_equal(msg0, msg)     # the error draws do not change the messages


def test_decode_packet_uncorrectable_path(oracle):
    """A segment whose syndrome names no position (s > n) makes the
    packet status 2, reports s, and leaves that segment as received (R15)."""
    M, t = 1, 1
    k, n, _ = oracle.packet_layout(8, 1)
    assert n == [12]
    msg = np.array([0xA7], np.uint8)
    bits = np.unpackbits(oracle.encode_packet(M, t, msg), bitorder="little")
    bits[12 - 1] ^= 1
    bits[1 - 1] ^= 1          # s = 12 ^ 1 = 13 > n = 12
    rx = np.packbits(bits, bitorder="little")
    out, syn, st = oracle.decode_packet(M, t, rx)
    assert int(syn[0]) == 13 and st == 2
    # as received: position 12 (data bit 7) flipped, position 1 is parity
    assert int(out[0]) == 0xA7 ^ 0x80
    # two segments: the clean one is still decoded, the packet still fails
    M, t = 4, 2
    k, n, _ = oracle.packet_layout(32, 2)
    msg = np.array([1, 2, 3, 4], np.uint8)
    bits = np.unpackbits(oracle.encode_packet(M, t, msg), bitorder="little")
    off = n[0]
    bits[off + 3 - 1] ^= 1
    bits[off + n[1] - 1] ^= 1   # s = 3 ^ n1
    s_exp = 3 ^ n[1]
    out, syn, st = oracle.decode_packet(M, t, np.packbits(bits, bitorder="little"))
    assert int(syn[0]) == 0 and int(syn[1]) == s_exp
    assert st == (2 if s_exp > n[1] else 1)
