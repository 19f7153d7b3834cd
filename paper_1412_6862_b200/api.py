"""Python binding of the C ABI (include/hamming.h), same names, on torch CUDA
tensors.  torch supplies device memory and streams only; every step of the
decode runs in libhamming.so's sm_100a kernels.

Readings of the paper used by the layout (R3, R4): LSB-first
packed streams; codeword c = stream bits [c*n, c*n + n); data bits of c at
[c*k, c*k + k).
"""
from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass
from typing import Optional

import torch

from ._lib import check, lib

TILE = 1024  # codewords per warp tile of the decode kernel


def code_nk(m: int) -> tuple[int, int]:
    """(n, k) of the perfect code of order m; decode takes m in [2, 8],
    encode / the synthetic channel m in [2, 6]."""
    if not 2 <= m <= 8:
        raise ValueError("m must be in [2, 8]")
    n = (1 << m) - 1
    return n, n - m


def coded_bytes(m: int, n_codewords: int) -> int:
    """ceil(n N / 8) -- the same value as the C ABI's hamming_coded_bytes (tested), computed here
    so the per-call path makes no extra foreign calls."""
    n, N = (1 << m) - 1, int(n_codewords)
    if not 2 <= m <= 8 or N > ((1 << 64) - 1) // n:
        return 0
    return (n * N + 7) >> 3


def data_bytes(m: int, n_codewords: int) -> int:
    """ceil(k N / 8), as hamming_data_bytes."""
    n, N = (1 << m) - 1, int(n_codewords)
    if not 2 <= m <= 8 or N > ((1 << 64) - 1) // n:
        return 0
    return ((n - m) * N + 7) >> 3


def channel_thresholds(p: float, q2: float) -> tuple[int, int, int]:
    """(thresh, all, q2thresh) of the synthetic channel: an error event iff
    u < floor(p 2^64) (all codewords when p >= 1); weight 2 iff
    hi32(u) < floor(q2 2^32)."""
    if not (0.0 <= p <= 1.0 and 0.0 <= q2 <= 1.0):
        raise ValueError("p and q2 must lie in [0, 1]")
    all_ = 1 if p >= 1.0 else 0
    return (0 if all_ else int(p * 2.0 ** 64)), all_, int(q2 * 2.0 ** 32)


def _dev_ptr(t: Optional[torch.Tensor], name: str, min_bytes: int):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.nbytes < min_bytes:
        raise ValueError(f"{name} holds {t.nbytes} bytes, needs {min_bytes}")
    return t.data_ptr()  # an int; the argtypes make it a void*


def _device_of(*tensors):
    """The one CUDA device all the given tensors (None skipped) live on."""
    dev = None
    for t in tensors:
        if t is None:
            continue
        if not t.is_cuda:
            raise ValueError("every device buffer must be a CUDA tensor")
        if dev is None:
            dev = t.device
        elif t.device != dev:
            raise ValueError(f"buffers on different devices: {dev} and {t.device}")
    return dev


def _on(dev):
    """Make `dev` current for the duration of a C-ABI call: the library launches on
    the current device, and the stream handle comes from `dev`.  No-op (no context
    switch) in the common case that it already is."""
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if torch.cuda.current_device() == idx:
        return contextlib.nullcontext()
    return torch.cuda.device(idx)


# torch's current raw cudaStream_t without building a Stream object (a few us per call on the
# latency-bound small-packet path); the public API is the fallback
_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_handle(stream, device):
    if stream is not None:
        return stream.cuda_stream
    if _raw_stream is not None:
        return _raw_stream(device.index if device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class DecodeResult:
    data: torch.Tensor                  # uint8 [data_bytes(m, N)]
    syndromes: Optional[torch.Tensor]   # uint8 [N] or None
    corrected: torch.Tensor             # int64 [1], device-resident count


def hamming_decode(m: int, rx: torch.Tensor, n_codewords: int, *, data_out: Optional[torch.Tensor] = None,
                   syndromes: bool | torch.Tensor = True, corrected: Optional[torch.Tensor] = None,
                   stream: Optional[torch.cuda.Stream] = None) -> DecodeResult:
    """Decode `n_codewords` (2^m-1, 2^m-1-m) codewords of the packed packet
    `rx` (uint8 CUDA tensor) -- include/hamming.h `hamming_decode`."""
    code_nk(m)
    N = int(n_codewords)
    dev = rx.device
    if data_out is None:
        data_out = torch.empty(max(1, data_bytes(m, N)), dtype=torch.uint8, device=dev)
    if syndromes is True:
        syn = torch.empty(max(1, N), dtype=torch.uint8, device=dev)
    elif syndromes is False or syndromes is None:
        syn = None
    else:
        syn = syndromes
    if corrected is None:
        corrected = torch.empty(1, dtype=torch.int64, device=dev)
    dev = _device_of(rx, data_out, syn, corrected)
    with _on(dev):
        st = lib().hamming_decode(m, _dev_ptr(rx, "rx", coded_bytes(m, N)), N,
                                  _dev_ptr(data_out, "data_out", data_bytes(m, N)),
                                  _dev_ptr(syn, "syndromes", N), _dev_ptr(corrected, "corrected", 8),
                                  _stream_handle(stream, dev))
    check(st, "hamming_decode")
    return DecodeResult(data_out, syn, corrected)


decode = hamming_decode


def hamming_encode(m: int, data: torch.Tensor, n_codewords: int, *, rx_out: Optional[torch.Tensor] = None,
                   stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    code_nk(m)
    N = int(n_codewords)
    if rx_out is None:
        rx_out = torch.empty(max(1, coded_bytes(m, N)), dtype=torch.uint8, device=data.device)
    dev = _device_of(data, rx_out)
    with _on(dev):
        st = lib().hamming_encode(m, _dev_ptr(data, "data", data_bytes(m, N)), N,
                                  _dev_ptr(rx_out, "rx_out", coded_bytes(m, N)), _stream_handle(stream, dev))
    check(st, "hamming_encode")
    return rx_out


encode = hamming_encode


def hamming_channel_generate(m: int, seed: int, c_first: int, n_codewords: int, p: float = 0.1, q2: float = 0.0,
                             *, rx_out: Optional[torch.Tensor] = None, device=None,
                             stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """Seeded synthetic received packet on the GPU."""
    code_nk(m)
    N = int(n_codewords)
    thresh, all_, q2t = channel_thresholds(p, q2)
    if rx_out is None:
        rx_out = torch.empty(max(1, coded_bytes(m, N)), dtype=torch.uint8,
                             device=device if device is not None else "cuda")
    dev = _device_of(rx_out)
    with _on(dev):
        st = lib().hamming_channel_generate(m, seed & (2 ** 64 - 1), c_first, N, thresh, all_, q2t,
                                            _dev_ptr(rx_out, "rx_out", coded_bytes(m, N)), _stream_handle(stream, dev))
    check(st, "hamming_channel_generate")
    return rx_out


channel_generate = hamming_channel_generate


def host_workspace_bytes(m: int, chunk_codewords: int, n_streams: int, with_syndromes: bool) -> int:
    return int(lib().hamming_host_workspace_bytes(m, chunk_codewords, n_streams, int(with_syndromes)))


def hamming_decode_host(m: int, rx_host: torch.Tensor, n_codewords: int, data_host: torch.Tensor,
                        syndromes_host: Optional[torch.Tensor], workspace: torch.Tensor,
                        chunk_codewords: int = 1 << 24, n_streams: int = 3) -> int:
    """End-to-end decode of a HOST packet (pinned CPU tensors) through the
    library's pipelined H2D / decode / D2H path (P:L113-132 ADT).  Returns the
    corrected count."""
    code_nk(m)
    N = int(n_codewords)
    for t, name in ((rx_host, "rx_host"), (data_host, "data_host"), (syndromes_host, "syndromes_host")):
        if t is not None and (t.is_cuda or not t.is_contiguous()):
            raise ValueError(f"{name} must be a contiguous CPU tensor")
    if rx_host.numel() < coded_bytes(m, N) or data_host.numel() < data_bytes(m, N):
        raise ValueError("host buffers too small")
    if syndromes_host is not None and syndromes_host.numel() < N:
        raise ValueError("syndromes_host too small")
    need = host_workspace_bytes(m, chunk_codewords, n_streams, syndromes_host is not None)
    if need == 0:
        raise ValueError("bad chunk_codewords / n_streams (1 <= n_streams <= 4)")
    dev = _device_of(workspace)
    cnt = ctypes.c_ulonglong(0)
    with _on(dev):
        # the library's streams do not wait on torch's: finish whatever still uses the workspace
        torch.cuda.current_stream(dev).synchronize()
        st = lib().hamming_decode_host(m, ctypes.c_void_p(rx_host.data_ptr()), N,
                                       ctypes.c_void_p(data_host.data_ptr()),
                                       None if syndromes_host is None else ctypes.c_void_p(syndromes_host.data_ptr()),
                                       ctypes.byref(cnt), _dev_ptr(workspace, "workspace", need), chunk_codewords,
                                       n_streams)
    check(st, "hamming_decode_host")
    return int(cnt.value)


decode_host = hamming_decode_host


def last_launch_count() -> int:
    return int(lib().hamming_last_launch_count())


def last_grid_blocks() -> int:
    return int(lib().hamming_last_grid_blocks())


# ------------------------------------------------ packets (the paper's workload)
def packet_layout(msg_bytes: int, t: int) -> tuple[list[int], list[int]]:
    """(seg_k, seg_n) of a msg_bytes-byte packet split into t segments."""
    k = (ctypes.c_uint32 * max(1, t))()
    n = (ctypes.c_uint32 * max(1, t))()
    check(lib().hamming_packet_layout(msg_bytes, t, k, n), "hamming_packet_layout")
    return list(k[:t]), list(n[:t])


def packet_coded_bytes(msg_bytes: int, t: int) -> int:
    v = int(lib().hamming_packet_coded_bytes(msg_bytes, t))
    if v == 0:
        raise ValueError("bad packet shape")
    return v


def packet_stride(msg_bytes: int, t: int) -> int:
    """The smallest legal rx_stride: coded bytes rounded up to 16."""
    return (packet_coded_bytes(msg_bytes, t) + 15) // 16 * 16


def packet_launch_shape(msg_bytes: int, t: int, n_packets: int, rx_stride: Optional[int] = None,
                        sm_count: int = 148) -> dict:
    """The launch shape hamming_decode_packets picks (host-only query, no CUDA call)."""
    rx_stride = packet_stride(msg_bytes, t) if rx_stride is None else rx_stride
    vals = [ctypes.c_int(0) for _ in range(5)]
    check(lib().hamming_packet_launch_shape(msg_bytes, t, rx_stride, int(n_packets), sm_count,
                                            *[ctypes.byref(v) for v in vals]), "hamming_packet_launch_shape")
    return dict(zip(("warps", "packets_per_batch", "lanes_per_item", "ctas_per_sm", "smem_bytes"),
                    (v.value for v in vals)))


@dataclass
class PacketDecodeResult:
    messages: torch.Tensor             # uint8 [n_packets * msg_stride]
    syndromes: Optional[torch.Tensor]  # uint16 as int16 storage [n_packets, t]
    status: Optional[torch.Tensor]     # uint8 [n_packets]: 0 clean, 1 corrected, 2 uncorrectable
    counts: torch.Tensor               # int64 [2]: segments corrected, segments uncorrectable


def hamming_decode_packets(msg_bytes: int, t: int, rx: torch.Tensor, n_packets: int, *, rx_stride: Optional[int] = None,
                           msg_out: Optional[torch.Tensor] = None, msg_stride: Optional[int] = None,
                           syndromes: bool = True, status: bool = True,
                           stream: Optional[torch.cuda.Stream] = None) -> PacketDecodeResult:
    rx_stride = packet_stride(msg_bytes, t) if rx_stride is None else rx_stride
    msg_stride = msg_bytes if msg_stride is None else msg_stride
    P = int(n_packets)
    dev = rx.device
    if msg_out is None:
        msg_out = torch.empty(max(1, P * msg_stride), dtype=torch.uint8, device=dev)
    syn = torch.empty((max(1, P), t), dtype=torch.int16, device=dev) if syndromes else None
    st = torch.empty(max(1, P), dtype=torch.uint8, device=dev) if status else None
    counts = torch.empty(2, dtype=torch.int64, device=dev)
    dev = _device_of(rx, msg_out, syn, st, counts)
    with _on(dev):
        rc = lib().hamming_decode_packets(msg_bytes, t, _dev_ptr(rx, "rx", rx_stride * P), rx_stride, P,
                                          _dev_ptr(msg_out, "msg_out", msg_stride * P), msg_stride,
                                          _dev_ptr(syn, "syndromes", 2 * t * P), _dev_ptr(st, "status", P),
                                          _dev_ptr(counts, "counts", 16), _stream_handle(stream, dev))
    check(rc, "hamming_decode_packets")
    return PacketDecodeResult(msg_out, syn, st, counts)


decode_packets = hamming_decode_packets


def hamming_encode_packets(msg_bytes: int, t: int, messages: torch.Tensor, n_packets: int, *,
                           msg_stride: Optional[int] = None, rx_stride: Optional[int] = None,
                           rx_out: Optional[torch.Tensor] = None,
                           stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    rx_stride = packet_stride(msg_bytes, t) if rx_stride is None else rx_stride
    msg_stride = msg_bytes if msg_stride is None else msg_stride
    P = int(n_packets)
    if rx_out is None:
        rx_out = torch.empty(max(1, P * rx_stride), dtype=torch.uint8, device=messages.device)
    dev = _device_of(messages, rx_out)
    with _on(dev):
        rc = lib().hamming_encode_packets(msg_bytes, t, _dev_ptr(messages, "messages", msg_stride * P), msg_stride,
                                          P, _dev_ptr(rx_out, "rx_out", rx_stride * P), rx_stride,
                                          _stream_handle(stream, dev))
    check(rc, "hamming_encode_packets")
    return rx_out


encode_packets = hamming_encode_packets


def hamming_packet_channel_generate(msg_bytes: int, t: int, seed: int, g_first: int, n_packets: int, p: float = 1.0,
                                    *, rx_stride: Optional[int] = None, want_messages: bool = False, device=None,
                                    stream: Optional[torch.cuda.Stream] = None):
    """Seeded received packets (one flip per segment with probability p).
    Returns (rx, messages|None)."""
    rx_stride = packet_stride(msg_bytes, t) if rx_stride is None else rx_stride
    P = int(n_packets)
    thresh, all_, _ = channel_thresholds(p, 0.0)
    device = device if device is not None else "cuda"
    rx = torch.empty(max(1, P * rx_stride), dtype=torch.uint8, device=device)
    msgs = torch.empty(max(1, P * msg_bytes), dtype=torch.uint8, device=device) if want_messages else None
    dev = _device_of(rx, msgs)
    with _on(dev):
        rc = lib().hamming_packet_channel_generate(msg_bytes, t, seed & (2 ** 64 - 1), g_first, P, thresh, all_,
                                                   _dev_ptr(rx, "rx", rx_stride * P), rx_stride,
                                                   _dev_ptr(msgs, "messages", msg_bytes * P),
                                                   _stream_handle(stream, dev))
    check(rc, "hamming_packet_channel_generate")
    return rx, msgs


packet_channel_generate = hamming_packet_channel_generate


# ------------------------------------------------------- SECDED (extended Hamming)
def secded_coded_bytes(m: int, n_codewords: int) -> int:
    v = int(lib().hamming_secded_coded_bytes(m, n_codewords))
    if n_codewords and v == 0:
        raise ValueError("SECDED needs m in [3, 6]")
    return v


@dataclass
class SecdedResult:
    data: torch.Tensor             # uint8 [data_bytes(m, N)]
    flags: Optional[torch.Tensor]  # uint8 [N]: s | 0x40 corrected | 0x80 double error detected
    counts: torch.Tensor           # int64 [2]: corrected, detected


def hamming_decode_secded(m: int, rx: torch.Tensor, n_codewords: int, *, data_out: Optional[torch.Tensor] = None,
                          flags: bool | torch.Tensor = True, counts: Optional[torch.Tensor] = None,
                          stream: Optional[torch.cuda.Stream] = None) -> SecdedResult:
    N = int(n_codewords)
    dev = rx.device
    if data_out is None:
        data_out = torch.empty(max(1, data_bytes(m, N)), dtype=torch.uint8, device=dev)
    if flags is True:
        fl = torch.empty(max(1, N), dtype=torch.uint8, device=dev)
    elif flags is False or flags is None:
        fl = None
    else:
        fl = flags
    if counts is None:
        counts = torch.empty(2, dtype=torch.int64, device=dev)
    dev = _device_of(rx, data_out, fl, counts)
    with _on(dev):
        st = lib().hamming_decode_secded(m, _dev_ptr(rx, "rx", secded_coded_bytes(m, N)), N,
                                         _dev_ptr(data_out, "data_out", data_bytes(m, N)), _dev_ptr(fl, "flags", N),
                                         _dev_ptr(counts, "counts", 16), _stream_handle(stream, dev))
    check(st, "hamming_decode_secded")
    return SecdedResult(data_out, fl, counts)


decode_secded = hamming_decode_secded


def hamming_encode_secded(m: int, data: torch.Tensor, n_codewords: int, *, rx_out: Optional[torch.Tensor] = None,
                          stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    N = int(n_codewords)
    if rx_out is None:
        rx_out = torch.empty(max(1, secded_coded_bytes(m, N)), dtype=torch.uint8, device=data.device)
    dev = _device_of(data, rx_out)
    with _on(dev):
        st = lib().hamming_encode_secded(m, _dev_ptr(data, "data", data_bytes(m, N)), N,
                                         _dev_ptr(rx_out, "rx_out", secded_coded_bytes(m, N)),
                                         _stream_handle(stream, dev))
    check(st, "hamming_encode_secded")
    return rx_out


encode_secded = hamming_encode_secded


def hamming_channel_generate_secded(m: int, seed: int, c_first: int, n_codewords: int, p: float = 0.1,
                                    q2: float = 0.0, *, device=None,
                                    stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    N = int(n_codewords)
    thresh, all_, q2t = channel_thresholds(p, q2)
    rx = torch.empty(max(1, secded_coded_bytes(m, N)), dtype=torch.uint8,
                     device=device if device is not None else "cuda")
    dev = _device_of(rx)
    with _on(dev):
        st = lib().hamming_channel_generate_secded(m, seed & (2 ** 64 - 1), c_first, N, thresh, all_, q2t,
                                                   _dev_ptr(rx, "rx", secded_coded_bytes(m, N)),
                                                   _stream_handle(stream, dev))
    check(st, "hamming_channel_generate_secded")
    return rx


channel_generate_secded = hamming_channel_generate_secded
