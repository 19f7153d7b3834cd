"""CPU oracle for the Hamming decoder of arXiv 1412.6862 (§II, §III.A,
Algorithm 1) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The
product path (``paper_1412_6862_b200``) never imports it and shares no code
with it; see ``oracle/oracle.c`` for the per-function paper citations.

This module is argument marshalling around ``liboracle.so`` (plain C, built
with ``gcc -O2``) plus a harness-level thread splitter for timing: the
per-codeword arithmetic stays the plain single-threaded C; threads only get
disjoint, 8-codeword-aligned ranges (so every range starts on a byte in
both the received and the data stream).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile ``liboracle.so`` with plain ``gcc -O2`` (no -march, no
    intrinsics).  Returns the library path."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-shared",
                               "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        u8p = ctypes.POINTER(ctypes.c_uint8)
        ip = ctypes.POINTER(ctypes.c_int)
        u64 = ctypes.c_uint64
        L.oracle_parity_bit_count.argtypes = [ctypes.c_int]
        L.oracle_parity_positions.argtypes = [ctypes.c_int]
        L.oracle_index_set.argtypes = [ctypes.c_int, ctypes.c_int, ip]
        L.oracle_syndrome_bits.argtypes = [ctypes.c_int, u8p]
        L.oracle_correct_bits.argtypes = [ctypes.c_int, u8p, ctypes.c_int]
        L.oracle_remove_redundancy_bits.argtypes = [ctypes.c_int, u8p, u8p]
        L.oracle_encode_bits.argtypes = [ctypes.c_int, u8p, u8p]
        L.oracle_decode.argtypes = [ctypes.c_int, ctypes.c_void_p, u64, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.POINTER(u64)]
        L.oracle_encode.argtypes = [ctypes.c_int, ctypes.c_void_p, u64, ctypes.c_void_p]
        L.oracle_generate.argtypes = [ctypes.c_int, u64, u64, u64, u64, ctypes.c_int, u64,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_count_events.argtypes = [u64, u64, u64, u64, ctypes.c_int, u64, ctypes.POINTER(u64),
                                          ctypes.POINTER(u64)]
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.oracle_packet_layout.argtypes = [ctypes.c_uint32, ctypes.c_int, u32p, u32p]
        L.oracle_packet_layout.restype = ctypes.c_long
        L.oracle_encode_packet.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_decode_packet.argtypes = [ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]
        L.oracle_generate_packets.argtypes = [ctypes.c_uint32, ctypes.c_int, u64, u64, u64, u64, ctypes.c_int,
                                              ctypes.c_void_p, u64, ctypes.c_void_p]
        L.oracle_decode_secded.argtypes = [ctypes.c_int, ctypes.c_void_p, u64, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.oracle_encode_secded.argtypes = [ctypes.c_int, ctypes.c_void_p, u64, ctypes.c_void_p]
        L.oracle_generate_secded.argtypes = [ctypes.c_int, u64, u64, u64, u64, ctypes.c_int, u64,
                                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        _lib = L
    return _lib


def _u8(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------- geometry
def code_nk(m: int) -> tuple[int, int]:
    n = (1 << m) - 1
    return n, n - m


def coded_bytes(m: int, count: int) -> int:
    n, _ = code_nk(m)
    return (n * count + 7) // 8


def data_bytes(m: int, count: int) -> int:
    _, k = code_nk(m)
    return (k * count + 7) // 8


def parity_bit_count(k: int) -> int:
    return lib().oracle_parity_bit_count(k)


def index_set(j: int, n: int) -> list[int]:
    out = (ctypes.c_int * n)()
    cnt = lib().oracle_index_set(j, n, out)
    if cnt < 0:
        raise ValueError(f"index_set: j={j} out of range for n={n}")
    return list(out[:cnt])


# ------------------------------------------------------- one codeword (bits)
def encode_bits(n: int, msg) -> np.ndarray:
    r = lib().oracle_parity_positions(n)
    msg = np.ascontiguousarray(msg, dtype=np.uint8)
    if msg.size != n - r:
        raise ValueError("encode_bits: message length != k")
    cw = np.zeros(n, np.uint8)
    lib().oracle_encode_bits(n, _u8(msg), _u8(cw))
    return cw


def syndrome_bits(n: int, bits) -> int:
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    if bits.size != n:
        raise ValueError("syndrome_bits: length != n")
    return lib().oracle_syndrome_bits(n, _u8(bits))


def correct_bits(n: int, bits, s: int) -> tuple[np.ndarray, int]:
    """Returns (corrected copy, status) with status 0 = unchanged,
    1 = flipped position s, -1 = uncorrectable (s > n)."""
    b = np.array(bits, dtype=np.uint8, copy=True)
    st = lib().oracle_correct_bits(n, _u8(b), s)
    return b, st


def remove_redundancy_bits(n: int, bits) -> np.ndarray:
    bits = np.ascontiguousarray(bits, dtype=np.uint8)
    msg = np.zeros(n, np.uint8)
    k = lib().oracle_remove_redundancy_bits(n, _u8(bits), _u8(msg))
    return msg[:k].copy()


# --------------------------------------------------------------- streams
def decode(m: int, rx: np.ndarray, count: int, want_syndromes: bool = True):
    """Single-threaded oracle decode.  Returns (data, syndromes|None, corrected)."""
    rx = np.ascontiguousarray(rx, dtype=np.uint8)
    if rx.size < coded_bytes(m, count):
        raise ValueError("decode: rx too short")
    # outputs start as 0xFF: the oracle must write every data bit and every pad bit itself
    data = np.full(data_bytes(m, count), 0xFF, np.uint8)
    syn = np.full(count, 0xFF, np.uint8) if want_syndromes else None
    cnt = ctypes.c_uint64(0)
    st = lib().oracle_decode(m, _ptr(rx), count, _ptr(data), _ptr(syn), ctypes.byref(cnt))
    if st != 0:
        raise RuntimeError(f"oracle_decode failed: {st}")
    return data, syn, int(cnt.value)


def _ranges(count: int, parts: int, align: int = 8):
    parts = max(1, parts)
    edges = [min(count, (count * i // parts) // align * align) for i in range(parts)] + [count]
    return [(a, b) for a, b in zip(edges[:-1], edges[1:]) if b > a]


def decode_mt(m: int, rx: np.ndarray, count: int, threads: int, want_syndromes: bool = True):
    """Harness-level parallel oracle decode: the same plain C routine run on
    disjoint 8-codeword-aligned ranges by `threads` OS threads (ctypes
    releases the GIL).  Bit-identical to decode()."""
    n, k = code_nk(m)
    rx = np.ascontiguousarray(rx, dtype=np.uint8)
    data = np.full(data_bytes(m, count), 0xFF, np.uint8)
    syn = np.full(count, 0xFF, np.uint8) if want_syndromes else None
    L = lib()

    def run(r):
        a, b = r
        cnt = ctypes.c_uint64(0)
        rxp = ctypes.c_void_p(rx.ctypes.data + a * n // 8)
        dp = ctypes.c_void_p(data.ctypes.data + a * k // 8)
        sp = None if syn is None else ctypes.c_void_p(syn.ctypes.data + a)
        st = L.oracle_decode(m, rxp, b - a, dp, sp, ctypes.byref(cnt))
        if st != 0:
            raise RuntimeError(f"oracle_decode failed: {st}")
        return int(cnt.value)

    with ThreadPoolExecutor(max(1, threads)) as ex:
        total = sum(ex.map(run, _ranges(count, threads)))
    return data, syn, total


def encode(m: int, data: np.ndarray, count: int) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    rx = np.zeros(coded_bytes(m, count), np.uint8)
    if lib().oracle_encode(m, _ptr(data), count, _ptr(rx)) != 0:
        raise RuntimeError("oracle_encode failed")
    return rx


def channel_thresholds(p: float, q2: float) -> tuple[int, int, int]:
    """(thresh, all, q2thresh) for oracle_generate: event iff u < floor(p 2^64)
    (or `all` when p >= 1); weight 2 iff hi32(u) < floor(q2 2^32)."""
    if not (0.0 <= p <= 1.0 and 0.0 <= q2 <= 1.0):
        raise ValueError("p and q2 must lie in [0, 1]")
    all_ = 1 if p >= 1.0 else 0
    thresh = 0 if all_ else int(p * 2.0 ** 64)
    q2t = int(q2 * 2.0 ** 32)
    return thresh, all_, q2t


def generate(m: int, seed: int, c_first: int, count: int, p: float = 0.1, q2: float = 0.0,
             want_sent: bool = False, want_err: bool = False, threads: int = 1):
    """Seeded synthetic packet: returns (rx, sent|None, err|None)."""
    n, k = code_nk(m)
    if c_first % 8 and threads > 1:
        raise ValueError("generate: threaded ranges need c_first % 8 == 0")
    thresh, all_, q2t = channel_thresholds(p, q2)
    rx = np.zeros(coded_bytes(m, count), np.uint8)
    sent = np.zeros(data_bytes(m, count), np.uint8) if want_sent else None
    err = np.zeros(2 * count, np.uint8) if want_err else None
    L = lib()

    def run(r):
        a, b = r
        rxp = ctypes.c_void_p(rx.ctypes.data + a * n // 8)
        sp = None if sent is None else ctypes.c_void_p(sent.ctypes.data + a * k // 8)
        ep = None if err is None else ctypes.c_void_p(err.ctypes.data + 2 * a)
        st = L.oracle_generate(m, seed & (2 ** 64 - 1), c_first + a, b - a, thresh, all_, q2t,
                               rxp, sp, ep)
        if st != 0:
            raise RuntimeError(f"oracle_generate failed: {st}")

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(run, _ranges(count, threads)))
    return rx, sent, err


def count_events(seed: int, c_first: int, count: int, p: float = 0.1, q2: float = 0.0, threads: int = 1):
    """(events, weight-2 events) of the seeded channel over global codewords
    c_first .. c_first + count - 1 -- the draws of generate() alone, for
    packets too large to generate on the host.  Independent of m."""
    thresh, all_, q2t = channel_thresholds(p, q2)
    L = lib()

    def run(r):
        a, b = r
        ev, w2 = ctypes.c_uint64(0), ctypes.c_uint64(0)
        L.oracle_count_events(seed & (2 ** 64 - 1), c_first + a, b - a, thresh, all_, q2t, ctypes.byref(ev),
                              ctypes.byref(w2))
        return int(ev.value), int(w2.value)

    with ThreadPoolExecutor(max(1, threads)) as ex:
        res = list(ex.map(run, _ranges(count, threads, align=1)))
    return sum(r[0] for r in res), sum(r[1] for r in res)


# ------------------------------------------------ packets (the paper's workload)
def packet_layout(msg_bits: int, t: int):
    """(seg_k, seg_n, total coded bits) -- near-equal split, larger first."""
    k = (ctypes.c_uint32 * max(1, t))()
    n = (ctypes.c_uint32 * max(1, t))()
    total = lib().oracle_packet_layout(msg_bits, t, k, n)
    if total < 0:
        raise ValueError(f"packet_layout: bad (msg_bits={msg_bits}, t={t})")
    return list(k[:t]), list(n[:t]), int(total)


def packet_coded_bytes(msg_bytes: int, t: int) -> int:
    return (packet_layout(msg_bytes * 8, t)[2] + 7) // 8


def encode_packet(msg_bytes: int, t: int, msg: np.ndarray) -> np.ndarray:
    msg = np.ascontiguousarray(msg, dtype=np.uint8)
    rx = np.zeros(packet_coded_bytes(msg_bytes, t), np.uint8)
    if lib().oracle_encode_packet(msg_bytes, t, _ptr(msg), _ptr(rx)) != 0:
        raise RuntimeError("oracle_encode_packet failed")
    return rx


def decode_packet(msg_bytes: int, t: int, rx: np.ndarray):
    """Returns (message bytes, syndromes[t] (uint16), status 0/1/2)."""
    rx = np.ascontiguousarray(rx, dtype=np.uint8)
    msg = np.zeros(msg_bytes, np.uint8)
    syn = np.zeros(t, np.uint16)
    st = lib().oracle_decode_packet(msg_bytes, t, _ptr(rx), _ptr(msg), _ptr(syn))
    if st < 0:
        raise RuntimeError("oracle_decode_packet failed")
    return msg, syn, int(st)


def generate_packets(msg_bytes: int, t: int, seed: int, g_first: int, count: int, stride: int,
                     p: float = 1.0, want_msg: bool = False, threads: int = 1):
    thresh, all_, _ = channel_thresholds(p, 0.0)
    rx = np.zeros(count * stride, np.uint8)
    msg = np.zeros(count * msg_bytes, np.uint8) if want_msg else None
    L = lib()

    def run(r):
        a, b = r
        rp = ctypes.c_void_p(rx.ctypes.data + a * stride)
        mp = None if msg is None else ctypes.c_void_p(msg.ctypes.data + a * msg_bytes)
        if L.oracle_generate_packets(msg_bytes, t, seed & (2 ** 64 - 1), g_first + a, b - a, thresh, all_,
                                     rp, stride, mp) != 0:
            raise RuntimeError("oracle_generate_packets failed")

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(run, _ranges(count, threads, align=1)))
    return rx, msg


def decode_packets(msg_bytes: int, t: int, rx: np.ndarray, count: int, stride: int, threads: int = 1):
    """Decode `count` packets `stride` bytes apart: (messages, syndromes[count, t], status[count])."""
    rx = np.ascontiguousarray(rx, dtype=np.uint8)
    msg = np.zeros(count * msg_bytes, np.uint8)
    syn = np.zeros((count, t), np.uint16)
    status = np.zeros(count, np.uint8)
    L = lib()

    def run(r):
        a, b = r
        for j in range(a, b):
            st = L.oracle_decode_packet(msg_bytes, t, ctypes.c_void_p(rx.ctypes.data + j * stride),
                                        ctypes.c_void_p(msg.ctypes.data + j * msg_bytes),
                                        ctypes.c_void_p(syn.ctypes.data + j * t * 2))
            if st < 0:
                raise RuntimeError("oracle_decode_packet failed")
            status[j] = st

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(run, _ranges(count, threads, align=1)))
    return msg, syn, status


# ------------------------------------------------------- SECDED (extended Hamming)
def secded_coded_bytes(m: int, count: int) -> int:
    return (count << m) // 8


def decode_secded(m: int, rx: np.ndarray, count: int):
    """Returns (data, flags[count] = s | 0x40 corrected | 0x80 double detected,
    corrected, detected)."""
    rx = np.ascontiguousarray(rx, dtype=np.uint8)
    data = np.full(data_bytes(m, count), 0xFF, np.uint8)
    flags = np.full(count, 0xFF, np.uint8)
    c1, c2 = ctypes.c_uint64(0), ctypes.c_uint64(0)
    if lib().oracle_decode_secded(m, _ptr(rx), count, _ptr(data), _ptr(flags), ctypes.byref(c1),
                                  ctypes.byref(c2)) != 0:
        raise RuntimeError("oracle_decode_secded failed")
    return data, flags, int(c1.value), int(c2.value)


def encode_secded(m: int, data: np.ndarray, count: int) -> np.ndarray:
    data = np.ascontiguousarray(data, dtype=np.uint8)
    rx = np.zeros(secded_coded_bytes(m, count), np.uint8)
    if lib().oracle_encode_secded(m, _ptr(data), count, _ptr(rx)) != 0:
        raise RuntimeError("oracle_encode_secded failed")
    return rx


def generate_secded(m: int, seed: int, c_first: int, count: int, p: float = 0.1, q2: float = 0.0,
                    want_sent: bool = False, want_err: bool = False):
    thresh, all_, q2t = channel_thresholds(p, q2)
    rx = np.zeros(secded_coded_bytes(m, count), np.uint8)
    sent = np.zeros(data_bytes(m, count), np.uint8) if want_sent else None
    err = np.zeros(2 * count, np.uint8) if want_err else None
    if lib().oracle_generate_secded(m, seed & (2 ** 64 - 1), c_first, count, thresh, all_, q2t, _ptr(rx),
                                    _ptr(sent), _ptr(err)) != 0:
        raise RuntimeError("oracle_generate_secded failed")
    return rx, sent, err
