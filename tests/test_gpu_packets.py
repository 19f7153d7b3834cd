"""GPU parity (-m gpu) for the paper's own workload:
packets of M message bytes split into t shortened-Hamming segments
 -- GPU decode/encode/generator against the CPU oracle,
bit for bit, including uncorrectable syndromes and miscorrections."""
import numpy as np
import pytest
import torch

import paper_1412_6862_b200 as ham

pytestmark = pytest.mark.gpu

GRID = [(M, t) for M in (400, 800, 1200, 1600, 2000) for t in (2, 3, 4, 5, 6)]
EDGE = [(1, 1), (1, 8), (13, 3), (16, 16), (1024, 1), (999, 7)]
# around the in-place head compaction threshold (every k >= 96): (12,1) k=96, (72,6) k=96,
# (71,6) k=94..95 (not compacted), (73,6) k=97..98, (97,8) k=97, (11,1) k=88
HEADX = [(12, 1), (72, 6), (71, 6), (73, 6), (97, 8), (11, 1)]


def gpu_decode(M, t, rx_np, P, stride):
    rx = torch.from_numpy(rx_np).cuda()
    res = ham.decode_packets(M, t, rx, P, rx_stride=stride)
    torch.cuda.synchronize()
    return (res.messages.cpu().numpy()[: P * M], res.syndromes.cpu().numpy().view(np.uint16)[:P],
            res.status.cpu().numpy()[:P], res.counts.cpu().numpy())


@pytest.mark.parametrize("M,t", GRID + EDGE)
def test_generator_matches_oracle(oracle, M, t):
    stride = ham.packet_stride(M, t)
    P = 37
    want, wmsg = oracle.generate_packets(M, t, 0xC0DE, 5, P, stride, p=0.7, want_msg=True)
    got, gmsg = ham.packet_channel_generate(M, t, 0xC0DE, 5, P, p=0.7, want_messages=True)
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy()[: P * stride], want)
    assert np.array_equal(gmsg.cpu().numpy()[: P * M], wmsg)


@pytest.mark.parametrize("M,t", GRID + EDGE + HEADX)
def test_decode_matches_oracle(oracle, M, t):
    stride = ham.packet_stride(M, t)
    P = 53
    rx, msg = oracle.generate_packets(M, t, 0xBEE + M + t, 0, P, stride, p=1.0, want_msg=True)
    wm, ws, wst = oracle.decode_packets(M, t, rx, P, stride)
    gm, gs, gst, cnt = gpu_decode(M, t, rx, P, stride)
    assert np.array_equal(gm, wm) and np.array_equal(gs, ws) and np.array_equal(gst, wst)
    assert np.array_equal(gm, msg)                       # one error per segment: all corrected
    assert cnt.tolist() == [int((ws > 0).sum()), 0]


@pytest.mark.parametrize("M,t", [(400, 2), (400, 6), (2000, 2), (13, 3), (1, 1), (16, 16), (999, 7)] + HEADX)
def test_random_received_packets(oracle, M, t):
    """Uniformly random received bits: many segments carry syndromes beyond
    n (uncorrectable) or miscorrect; GPU and oracle must agree exactly."""
    stride = ham.packet_stride(M, t)
    P = 64
    rng = np.random.default_rng(M * 31 + t)
    rx = rng.integers(0, 256, P * stride, dtype=np.uint8)
    cb = ham.packet_coded_bytes(M, t)
    wm, ws, wst = oracle.decode_packets(M, t, rx, P, stride)
    gm, gs, gst, cnt = gpu_decode(M, t, rx, P, stride)
    assert np.array_equal(gm, wm) and np.array_equal(gs, ws) and np.array_equal(gst, wst)
    k, n = ham.packet_layout(M, t)
    n = np.array(n)
    assert cnt.tolist() == [int(((ws > 0) & (ws <= n)).sum()), int((ws > n).sum())]
    if t <= 6 and M >= 400:
        assert (wst == 2).any()   # the uncorrectable path is exercised


@pytest.mark.parametrize("M,t", [(400, 3), (2000, 6), (13, 3), (4096, 16)])
def test_encode_matches_oracle(oracle, M, t):
    stride = ham.packet_stride(M, t)
    P = 20
    rng = np.random.default_rng(M + t)
    msgs = rng.integers(0, 256, P * M, dtype=np.uint8)
    got = ham.encode_packets(M, t, torch.from_numpy(msgs).cuda(), P).cpu().numpy()
    cb = ham.packet_coded_bytes(M, t)
    for j in range(P):
        if oracle.packet_layout(8 * M, t)[1][0] <= 16384:
            want = oracle.encode_packet(M, t, msgs[j * M:(j + 1) * M])
            assert np.array_equal(got[j * stride: j * stride + cb], want)
        assert not got[j * stride + cb:(j + 1) * stride].any()
    gm, gs, gst, cnt = gpu_decode(M, t, got, P, stride)
    assert np.array_equal(gm, msgs) and not gs.any() and not gst.any()


def test_strided_messages_and_no_outputs():
    M, t, P = 400, 4, 10
    rx, msg = ham.packet_channel_generate(M, t, 1, 0, P, p=1.0, want_messages=True)
    out = torch.zeros(P * 512, dtype=torch.uint8, device="cuda")
    res = ham.decode_packets(M, t, rx, P, msg_out=out, msg_stride=512, syndromes=False, status=False)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(P, 512)
    assert np.array_equal(o[:, :M].reshape(-1), msg.cpu().numpy()[: P * M]) and not o[:, M:].any()
    assert res.counts.cpu().tolist() == [P * t, 0]


@pytest.mark.parametrize("M,t", [(2048, 1), (4096, 1), (4096, 16), (4096, 5)])
def test_longest_segments_roundtrip(M, t):
    """Segments beyond the oracle's size limit (n up to 32784): encode -> one
    flip per segment -> decode recovers every message (closed-form check)."""
    P = 16
    rx, msg = ham.packet_channel_generate(M, t, 77, 0, P, p=1.0, want_messages=True)
    res = ham.decode_packets(M, t, rx, P)
    torch.cuda.synchronize()
    assert torch.equal(res.messages[: P * M], msg[: P * M])
    assert (res.status[:P] == 1).all() and res.counts.cpu().tolist() == [P * t, 0]


def _random_geometries(count, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < count:
        M = int(rng.choice([int(rng.integers(1, 64)), int(rng.integers(64, 1100)), int(rng.integers(1100, 4097))]))
        t = int(rng.integers(1, 17))
        if 8 * M < t:
            continue
        k0, n0 = ham.packet_layout(M, t)
        if max(n0) > 16384:      # the oracle's segment limit (larger ones: test_longest_segments_roundtrip)
            continue
        out.append((M, t, int(rng.integers(0, 3))))
    return out


@pytest.mark.parametrize("M,t,extra", _random_geometries(40, 0x9E0))
def test_random_geometries_strides_and_batches(oracle, M, t, extra):
    """Seeded random (M, t) over the whole accepted range, a received-packet
    stride padded by 0..2 extra 16-byte slots, random received bits plus
    encoded packets with single errors, a packet count that leaves a ragged
    last batch: messages, syndromes, statuses and counts equal the oracle's."""
    stride = ham.packet_stride(M, t) + 16 * extra
    P = 37 + 5 * extra
    rng = np.random.default_rng(M * 131 + t)
    rx, _ = oracle.generate_packets(M, t, 0xA11 + M, 0, P, stride, p=0.8, want_msg=True)
    noise = rng.integers(0, 256, P * stride, dtype=np.uint8)
    mix = np.where(np.repeat(rng.random(P) < 0.3, stride), noise, rx).astype(np.uint8)
    wm, ws, wst = oracle.decode_packets(M, t, mix, P, stride)
    gm, gs, gst, cnt = gpu_decode(M, t, mix, P, stride)
    assert np.array_equal(gm, wm) and np.array_equal(gs, ws) and np.array_equal(gst, wst)
    k, n = ham.packet_layout(M, t)
    n = np.array(n)
    assert cnt.tolist() == [int(((ws > 0) & (ws <= n)).sum()), int((ws > n).sum())]


@pytest.mark.parametrize("M,t", [(400, 5), (800, 3), (1200, 6), (2000, 2), (97, 8), (11, 1)])
def test_many_packets_multi_round(oracle, M, t):
    """200k packets: every warp of the persistent grid walks many batches and
    reuses its TMA stages and message buffer (the small tests stay in the first
    round).  One error per segment (the paper's regime): every message must come
    back as sent (the GPU generator is checked against the oracle above), the
    counts must be [P t, 0] and every status 1; three windows of packets are
    checked against the oracle byte for byte, syndromes included."""
    P = 200_000
    stride = ham.packet_stride(M, t)
    rx, sent = ham.packet_channel_generate(M, t, 0x5EED, 0, P, p=1.0, want_messages=True)
    res = ham.decode_packets(M, t, rx, P)
    torch.cuda.synchronize()
    msgs = res.messages.cpu().numpy()[: P * M]
    assert np.array_equal(msgs, sent.cpu().numpy()[: P * M])
    assert res.counts.cpu().numpy().tolist() == [P * t, 0]
    assert (res.status.cpu().numpy()[:P] == 1).all()
    rx_np = rx.cpu().numpy()
    syn = res.syndromes.cpu().numpy().view(np.uint16)[: P * t].reshape(P, t)
    for p0 in (0, P // 2 - 7, P - 300):
        cnt = 300
        wm, ws, wst = oracle.decode_packets(M, t, rx_np[p0 * stride:(p0 + cnt) * stride], cnt, stride)
        assert np.array_equal(msgs[p0 * M:(p0 + cnt) * M], wm)
        assert np.array_equal(syn[p0:p0 + cnt].reshape(-1), ws.reshape(-1))


@pytest.mark.parametrize("M,t,msg_stride", [(1200, 3, 1216), (1201, 5, 1201), (400, 6, 404), (2000, 2, 4096)])
def test_in_place_messages_with_word_and_byte_stores(M, t, msg_stride):
    """The head-compacted path writes messages in place over the input stage and
    refills a stage only after its stores have read it.  With a strided or
    unaligned message layout the stores are lane stores instead of TMA bulk
    stores: many batches per warp, every message back as sent, the gap bytes
    between strided messages untouched."""
    P = 30_000
    rx, sent = ham.packet_channel_generate(M, t, 0xBEE, 0, P, p=1.0, want_messages=True)
    out = torch.full((P * msg_stride,), 0xA5, dtype=torch.uint8, device="cuda")
    res = ham.decode_packets(M, t, rx, P, msg_out=out, msg_stride=msg_stride)
    torch.cuda.synchronize()
    o = out.cpu().numpy().reshape(P, msg_stride)
    assert np.array_equal(o[:, :M].reshape(-1), sent.cpu().numpy()[: P * M])
    assert (o[:, M:] == 0xA5).all()
    assert res.counts.cpu().tolist() == [P * t, 0] and bool((res.status[:P] == 1).all())


def test_counts_overwritten_without_memset_eager_and_in_graph(oracle):
    """The decoder writes its two counts itself (one CTA: stored; several: the last CTA publishes
    through the stream's launch slot; under graph capture: memset + atomics) -- repeated calls
    overwrite, never accumulate, on every path."""
    M, t = 400, 5
    stride = ham.packet_stride(M, t)
    for P in (3, 5000):  # one CTA / many CTAs
        rx_np, _ = oracle.generate_packets(M, t, 0xACE, 0, P, stride, p=0.6, want_msg=True)
        _, ws, _ = oracle.decode_packets(M, t, rx_np, P, stride)
        want = [int((ws != 0).sum()), 0]  # one flip per segment at most: every nonzero syndrome corrected
        rx = torch.from_numpy(rx_np).cuda()
        for _ in range(3):
            res = ham.decode_packets(M, t, rx, P, rx_stride=stride)
            torch.cuda.synchronize()
            assert res.counts.cpu().tolist() == want, P
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            out = torch.empty(P * M, dtype=torch.uint8, device="cuda")
            r0 = ham.decode_packets(M, t, rx, P, rx_stride=stride, msg_out=out, stream=side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=side):
                r1 = ham.decode_packets(M, t, rx, P, rx_stride=stride, msg_out=out, stream=side)
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
            torch.cuda.synchronize()
            assert r1.counts.cpu().tolist() == want, ("graph", P)
        assert r0.counts.cpu().tolist() == want
