"""C-ABI boundary checks that need no GPU (-m "not gpu"): the library loads,
exports every symbol include/hamming.h declares, its size helpers are right,
and argument validation returns before any CUDA call (fake pointers are fine
because nothing is dereferenced or launched)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_1412_6862_b200 as ham
from paper_1412_6862_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_1412_6862_b200 import build
    build.build()
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    declared = _lib.declared_functions()
    assert "hamming_decode" in declared and len(declared) >= 10
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (hamming_\w+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    for f in declared:
        getattr(L, f)


def test_library_is_sm100a_only(L):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_abi_and_sizes(L):
    assert L.hamming_abi_version() == 1
    for m in range(2, 9):
        n = 2 ** m - 1
        k = n - m
        for N in (0, 1, 7, 8, 1023, 1024, 4681, 10 ** 12):
            assert ham.coded_bytes(m, N) == (n * N + 7) // 8
            assert ham.data_bytes(m, N) == (k * N + 7) // 8
    assert ham.coded_bytes(9, 10) == 0 and ham.coded_bytes(1, 10) == 0
    assert ham.coded_bytes(6, 2 ** 64 // 63 + 1) == 0      # overflow
    # the binding computes the sizes in Python: the same values as the C ABI's helpers
    for m in (1, 2, 3, 6, 8, 9):
        for N in (0, 1, 4681, 10 ** 12, 2 ** 64 // 63, 2 ** 64 // 63 + 1, 2 ** 64 // 255 + 1):
            N = min(N, 2 ** 64 - 1)
            assert ham.coded_bytes(m, N) == L.hamming_coded_bytes(m, N), (m, N)
            assert ham.data_bytes(m, N) == L.hamming_data_bytes(m, N), (m, N)
    # the north-star shapes: a 4 KB (7,4) packet is 4681 codewords
    assert ham.coded_bytes(3, 4681) == 4096


def test_status_strings(L):
    for s in range(0, 8):
        assert L.hamming_status_string(s)


FAKE = 0x7F0000000000  # 16-byte aligned, never dereferenced


def _call_decode(L, m, rx, N, data, syn, cnt):
    return L.hamming_decode(m, ctypes.c_void_p(rx) if rx else None, N, ctypes.c_void_p(data) if data else None,
                            ctypes.c_void_p(syn) if syn else None, ctypes.c_void_p(cnt) if cnt else None, None)


def test_decode_argument_validation(L):
    big = 1 << 30
    assert _call_decode(L, 9, FAKE, 10, FAKE + big, FAKE + 2 * big, FAKE + 3 * big) == 1
    assert _call_decode(L, 1, FAKE, 10, FAKE + big, FAKE + 2 * big, FAKE + 3 * big) == 1
    assert _call_decode(L, 6, 0, 10, FAKE + big, 0, FAKE + 3 * big) == 2
    assert _call_decode(L, 6, FAKE, 10, 0, 0, FAKE + 3 * big) == 2
    assert _call_decode(L, 6, FAKE, 10, FAKE + big, 0, 0) == 2
    assert _call_decode(L, 6, FAKE + 4, 10, FAKE + big, 0, FAKE + 3 * big) == 3
    assert _call_decode(L, 6, FAKE, 10, FAKE + big + 8, 0, FAKE + 3 * big) == 3
    assert _call_decode(L, 6, FAKE, 10, FAKE + big, FAKE + 2 * big + 1, FAKE + 3 * big) == 3
    # rx [FAKE, FAKE+79) and data at FAKE+64 overlap
    assert _call_decode(L, 6, FAKE, 10, FAKE + 64, 0, FAKE + 3 * big) == 4
    assert _call_decode(L, 6, FAKE, 10, FAKE + big, FAKE + 32, FAKE + 3 * big) == 4
    assert _call_decode(L, 6, FAKE, 2 ** 64 // 63 + 1, FAKE + big, 0, FAKE + 3 * big) == 5
    assert b"overlap" in L.hamming_last_error() or b"overflow" in L.hamming_last_error()


def test_other_entry_point_validation(L):
    assert L.hamming_encode(9, None, 5, None, None) == 1
    assert L.hamming_encode(7, None, 5, None, None) == 1      # encode stops at m = 6
    assert L.hamming_encode(3, None, 5, None, None) == 2
    assert L.hamming_encode(3, ctypes.c_void_p(FAKE + 1), 5, ctypes.c_void_p(FAKE + (1 << 20)), None) == 3
    assert L.hamming_channel_generate(3, 1, 0, 5, 0, 0, 2 ** 32 + 1, ctypes.c_void_p(FAKE), None) == 5
    assert L.hamming_channel_generate(3, 1, 0, 5, 0, 0, 0, None, None) == 2
    assert L.hamming_host_workspace_bytes(6, 1024, 0, 1) == 0
    assert L.hamming_host_workspace_bytes(6, 1024, 2, 1) == 256 + 2 * (8192 + 7424 + 1024)
    cnt = ctypes.c_ulonglong()
    assert L.hamming_decode_host(6, None, 10, None, None, ctypes.byref(cnt), ctypes.c_void_p(FAKE), 1024, 2) == 2
    assert L.hamming_decode_host(6, ctypes.c_void_p(FAKE), 10, ctypes.c_void_p(FAKE), None, ctypes.byref(cnt),
                                 ctypes.c_void_p(FAKE), 1000, 2) == 7


def test_python_binding_rejects_cpu_tensors(L):
    import torch
    rx = torch.zeros(100, dtype=torch.uint8)
    with pytest.raises(ValueError):
        ham.decode(6, rx, 10, data_out=torch.zeros(100, dtype=torch.uint8), syndromes=False,
                   corrected=torch.zeros(1, dtype=torch.int64))


def test_product_package_never_touches_the_oracle():
    pkg = os.path.join(ROOT, "paper_1412_6862_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f), encoding="utf-8").read()
                assert not re.search(r"^\s*(import|from)\s+oracle", text, re.M), f
                assert "liboracle" not in text, f
                assert "oracle.c" not in text or f.endswith(".cu"), f


def test_packet_entry_point_validation(L):
    assert L.hamming_packet_coded_bytes(0, 2) == 0
    assert L.hamming_packet_coded_bytes(400, 0) == 0
    assert L.hamming_packet_coded_bytes(400, 17) == 0
    assert L.hamming_packet_coded_bytes(4097, 2) == 0
    assert L.hamming_packet_coded_bytes(2000, 2) == (2 * 8013 + 7) // 8
    cb = ham.packet_coded_bytes(400, 3)
    stride = ham.packet_stride(400, 3)
    assert stride % 16 == 0 and stride >= cb
    big = 1 << 30
    # stride too small / not a multiple of 16 / misaligned / NULL / overlap
    assert L.hamming_decode_packets(400, 3, ctypes.c_void_p(FAKE), 16, 4, ctypes.c_void_p(FAKE + big), 400,
                                    None, None, None, None) == 7
    assert L.hamming_decode_packets(400, 3, ctypes.c_void_p(FAKE), stride + 8, 4, ctypes.c_void_p(FAKE + big), 400,
                                    None, None, None, None) == 7
    assert L.hamming_decode_packets(400, 3, ctypes.c_void_p(FAKE + 8), stride, 4, ctypes.c_void_p(FAKE + big), 400,
                                    None, None, None, None) == 3
    assert L.hamming_decode_packets(400, 3, ctypes.c_void_p(FAKE), stride, 4, None, 400, None, None, None, None) == 2
    assert L.hamming_decode_packets(400, 3, ctypes.c_void_p(FAKE), stride, 4, ctypes.c_void_p(FAKE + 64), 400,
                                    None, None, None, None) == 4
    assert L.hamming_decode_packets(400, 3, ctypes.c_void_p(FAKE), stride, 4, ctypes.c_void_p(FAKE + big), 399,
                                    None, None, None, None) == 7


def test_secded_entry_point_validation(L):
    assert L.hamming_secded_coded_bytes(6, 1000) == 8000
    assert L.hamming_secded_coded_bytes(3, 8) == 8
    assert L.hamming_secded_coded_bytes(2, 8) == 0 and L.hamming_secded_coded_bytes(7, 8) == 0
    big = 1 << 30
    assert L.hamming_decode_secded(2, ctypes.c_void_p(FAKE), 8, ctypes.c_void_p(FAKE + big), None,
                                   ctypes.c_void_p(FAKE + 2 * big), None) == 1
    assert L.hamming_decode_secded(6, ctypes.c_void_p(FAKE), 8, ctypes.c_void_p(FAKE + big), None, None, None) == 2
    assert L.hamming_decode_secded(6, ctypes.c_void_p(FAKE + 4), 8, ctypes.c_void_p(FAKE + big), None,
                                   ctypes.c_void_p(FAKE + 2 * big), None) == 3
    assert L.hamming_decode_secded(6, ctypes.c_void_p(FAKE), 8, ctypes.c_void_p(FAKE + 32), None,
                                   ctypes.c_void_p(FAKE + 2 * big), None) == 4
    assert L.hamming_encode_secded(6, None, 8, None, None) == 2
    assert L.hamming_channel_generate_secded(6, 1, 0, 8, 0, 0, 2 ** 32 + 1, ctypes.c_void_p(FAKE), None) == 5
