"""Pins for the oracle's seeded input generators written from the recipe's
text in plain Python integers -- an independent
re-derivation of every draw, so a mistake in oracle.c's draw indices, keys,
thresholds or position formulas fails here:

  * the per-codeword channel (oracle_generate / oracle_count_events):
    u(c, q) = mix(seed + (4c + q + 1) gamma);
  * the packet channel (oracle_generate_packets, the paper's "one error per
    segment" regime): key = mix(seed + (g + 1) gamma),
    u(g, q) = mix(key + (q + 1) gamma), message byte b = byte (b & 7) of
    u(g, b >> 3), segment i's event draw u(g, W + 2i), position draw
    u(g, W + 2i + 1), flip at 1 + umulhi(lo32, n_i).

The Python splitmix64 is itself pinned to the public reference vectors."""
import json
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MASK = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix(z: int) -> int:
    """splitmix64 output function (Steele, Lea & Flood 2014)."""
    z &= MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
    return z ^ (z >> 31)


def u(seed: int, c: int, q: int) -> int:
    return mix(seed + (4 * c + q + 1) * GAMMA)


def test_python_splitmix_matches_reference_vectors():
    with open(os.path.join(GOLDEN, "splitmix64_vectors.json")) as f:
        g = json.load(f)
    state = g["seed"]
    for out in g["outputs"]:
        state = (state + GAMMA) & MASK
        assert mix(state) == int(out, 16)


@pytest.mark.parametrize("p,q2", [(0.1, 0.0), (0.3, 0.25), (1.0, 0.5), (0.0, 0.0)])
def test_count_events_rederived(oracle, p, q2):
    seed, c0, N = 0x14126862 ^ 5, 8_726_282_760 - 3000, 3000   # the tail of C5's index range
    thresh, all_, q2t = oracle.channel_thresholds(p, q2)
    ev = w2 = 0
    for c in range(c0, c0 + N):
        if all_ or u(seed, c, 1) < thresh:
            ev += 1
            w2 += (u(seed, c, 2) >> 32) < q2t
    assert oracle.count_events(seed, c0, N, p=p, q2=q2) == (ev, w2)
    assert oracle.count_events(seed, c0, N, p=p, q2=q2, threads=7) == (ev, w2)
    # and it agrees with the events oracle_generate records (same draws)
    _, _, err = oracle.generate(6, seed, c0, N, p=p, q2=q2, want_err=True)
    e = err.reshape(N, 2)
    assert int((e[:, 0] > 0).sum()) == ev and int((e[:, 1] > 0).sum()) == w2


@pytest.mark.parametrize("m", [3, 6])
def test_channel_draws_rederived(oracle, m):
    """Message bits and flip positions of oracle_generate, from the recipe."""
    n, k = oracle.code_nk(m)
    seed, c0, N, p, q2 = 0xBEEF, 1 << 33, 400, 0.5, 0.5
    thresh, all_, q2t = oracle.channel_thresholds(p, q2)
    _, sent, err = oracle.generate(m, seed, c0, N, p=p, q2=q2, want_sent=True, want_err=True)
    sent_bits = np.unpackbits(sent, bitorder="little")
    e = err.reshape(N, 2)
    for i in range(N):
        c = c0 + i
        msg = u(seed, c, 0) & ((1 << k) - 1)
        got = sum(int(b) << j for j, b in enumerate(sent_bits[i * k:(i + 1) * k]))
        assert got == msg
        p1 = p2 = 0
        if all_ or u(seed, c, 1) < thresh:
            w = u(seed, c, 3)
            p1 = 1 + (((w & 0xFFFFFFFF) * n) >> 32)
            if (u(seed, c, 2) >> 32) < q2t:
                p2 = 1 + ((p1 - 1 + 1 + (((w >> 32) * (n - 1)) >> 32)) % n)
        assert (int(e[i, 0]), int(e[i, 1])) == (p1, p2), i


@pytest.mark.parametrize("M,t,p", [(400, 5, 1.0), (13, 3, 0.5), (2000, 2, 0.7)])
def test_packet_channel_draws_rederived(oracle, M, t, p):
    """oracle_generate_packets: messages and the flipped position of every
    segment, re-derived from the recipe (the flip is recovered as received
    XOR the oracle's re-encoding of the sent message)."""
    k, n, total = oracle.packet_layout(8 * M, t)
    stride = (oracle.packet_coded_bytes(M, t) + 15) // 16 * 16
    seed, g0, P = 0x5EED, 1 << 40, 6
    thresh, all_, _ = oracle.channel_thresholds(p, 0.0)
    rx, msg = oracle.generate_packets(M, t, seed, g0, P, stride, p=p, want_msg=True)
    W = (M + 7) // 8
    flips_seen = 0
    for j in range(P):
        key = mix(seed + (g0 + j + 1) * GAMMA)
        ug = [mix(key + (q + 1) * GAMMA) for q in range(W + 2 * t)]
        want_msg = bytes((ug[b >> 3] >> (8 * (b & 7))) & 0xFF for b in range(M))
        assert msg[j * M:(j + 1) * M].tobytes() == want_msg
        clean = oracle.encode_packet(M, t, np.frombuffer(want_msg, np.uint8))
        got = rx[j * stride:(j + 1) * stride]
        diff = np.unpackbits(got[: clean.size] ^ clean, bitorder="little")
        assert not got[clean.size:].any()                      # pad bytes of the stride are 0
        off = 0
        for i in range(t):
            seg = np.nonzero(diff[off:off + n[i]])[0]
            if all_ or ug[W + 2 * i] < thresh:
                pos = 1 + (((ug[W + 2 * i + 1] & 0xFFFFFFFF) * n[i]) >> 32)
                assert seg.tolist() == [pos - 1], (j, i)
                flips_seen += 1
            else:
                assert seg.size == 0, (j, i)
            off += n[i]
        assert not diff[off:].any()
    assert flips_seen > 0
