"""Host logic of the packet decoder's launch shape (hamming_packet_launch_shape,
no CUDA call): over the paper's grid (M = 400..2000 B, t = 2..6) and
odd shapes, the chosen (warps, packets per batch, lanes per item) must be legal
for the kernel and fit the SM's shared memory; bad strides are rejected."""
import pytest

import paper_1412_6862_b200 as ham
from paper_1412_6862_b200._lib import HammingArgumentError

SMEM_SM = 228 * 1024


@pytest.mark.parametrize("M", [400, 800, 1200, 1600, 2000])
@pytest.mark.parametrize("t", [2, 3, 4, 5, 6])
def test_paper_grid_shapes_are_legal(M, t):
    for P in (1, 37, 1 << 19):
        s = ham.packet_launch_shape(M, t, P)
        assert 1 <= s["warps"] <= 16
        assert 1 <= s["packets_per_batch"] <= 64
        assert s["lanes_per_item"] in (1, 2, 4, 8, 16, 32)
        assert s["ctas_per_sm"] >= 1 and s["ctas_per_sm"] * s["warps"] <= 32  # 64 registers per thread
        assert s["smem_bytes"] <= 227 * 1024
        assert s["ctas_per_sm"] * (s["smem_bytes"] + 1536) <= SMEM_SM
        # a batch holds both TMA stages of its packets
        assert s["smem_bytes"] >= s["warps"] * 2 * s["packets_per_batch"] * ham.packet_stride(M, t)


def test_shape_is_deterministic_and_uses_the_sm_count():
    a = ham.packet_launch_shape(1200, 5, 1 << 19)
    assert a == ham.packet_launch_shape(1200, 5, 1 << 19)
    ham.packet_launch_shape(1200, 5, 1 << 19, sm_count=1)  # any positive SM count is accepted


@pytest.mark.parametrize("M,t", [(13, 3), (71, 6), (97, 8), (4096, 16), (4096, 1)])
def test_odd_shapes_and_padded_strides(M, t):
    st = ham.packet_stride(M, t)
    for stride in (st, st + 16, st + 4096):
        s = ham.packet_launch_shape(M, t, 1000, rx_stride=stride)
        assert s["smem_bytes"] <= 227 * 1024 and s["warps"] >= 1


def test_bad_strides_rejected():
    st = ham.packet_stride(400, 5)
    with pytest.raises(HammingArgumentError):
        ham.packet_launch_shape(400, 5, 10, rx_stride=st - 16)
    with pytest.raises(HammingArgumentError):
        ham.packet_launch_shape(400, 5, 10, rx_stride=st + 8)
    with pytest.raises(HammingArgumentError):
        ham.packet_launch_shape(400, 5, 10, rx_stride=200 * 1024)  # too large to stage
