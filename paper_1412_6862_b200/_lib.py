"""ctypes loader for ``libhamming.so`` (the C ABI in include/hamming.h).

Argument marshalling only.  There is no fallback: if the library or a CUDA
device is missing, calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os
import re

_PKG = os.path.dirname(os.path.abspath(__file__))
# HAMMING_LIB points the binding at another build of the same source (launch-shape
# tuning sweeps, tools/tune_shapes.sh); the default is the in-tree library.
LIB_PATH = os.environ.get("HAMMING_LIB") or os.path.join(_PKG, "libhamming.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "hamming.h")

STATUS = {
    0: "HAMMING_OK", 1: "HAMMING_E_INVALID_M", 2: "HAMMING_E_NULL", 3: "HAMMING_E_MISALIGNED",
    4: "HAMMING_E_OVERLAP", 5: "HAMMING_E_RANGE", 6: "HAMMING_E_CUDA", 7: "HAMMING_E_ARG",
}

_lib = None


class HammingError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {detail}")
        self.status = status


class HammingArgumentError(HammingError, ValueError):
    pass


def declared_functions() -> list[str]:
    """Every function name the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hamming_[a-z0-9_]+)\s*\(", text)))


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_1412_6862_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u64, c_int = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
    L.hamming_decode.argtypes = [c_int, vp, u64, vp, vp, vp, vp]
    L.hamming_decode.restype = c_int
    L.hamming_encode.argtypes = [c_int, vp, u64, vp, vp]
    L.hamming_encode.restype = c_int
    L.hamming_channel_generate.argtypes = [c_int, u64, u64, u64, u64, c_int, u64, vp, vp]
    L.hamming_channel_generate.restype = c_int
    L.hamming_host_workspace_bytes.argtypes = [c_int, u64, c_int, c_int]
    L.hamming_host_workspace_bytes.restype = ctypes.c_size_t
    L.hamming_decode_host.argtypes = [c_int, vp, u64, vp, vp, vp, vp, u64, c_int]
    L.hamming_decode_host.restype = c_int
    u32 = ctypes.c_uint32
    L.hamming_secded_coded_bytes.argtypes = [c_int, u64]
    L.hamming_secded_coded_bytes.restype = u64
    L.hamming_decode_secded.argtypes = [c_int, vp, u64, vp, vp, vp, vp]
    L.hamming_decode_secded.restype = c_int
    L.hamming_encode_secded.argtypes = [c_int, vp, u64, vp, vp]
    L.hamming_encode_secded.restype = c_int
    L.hamming_channel_generate_secded.argtypes = [c_int, u64, u64, u64, u64, c_int, u64, vp, vp]
    L.hamming_channel_generate_secded.restype = c_int
    L.hamming_packet_coded_bytes.argtypes = [u32, c_int]
    L.hamming_packet_coded_bytes.restype = u64
    L.hamming_packet_layout.argtypes = [u32, c_int, vp, vp]
    L.hamming_packet_layout.restype = c_int
    L.hamming_packet_launch_shape.argtypes = [u32, c_int, u64, u64, c_int, vp, vp, vp, vp, vp]
    L.hamming_packet_launch_shape.restype = c_int
    L.hamming_decode_packets.argtypes = [u32, c_int, vp, u64, u64, vp, u64, vp, vp, vp, vp]
    L.hamming_decode_packets.restype = c_int
    L.hamming_encode_packets.argtypes = [u32, c_int, vp, u64, u64, vp, u64, vp]
    L.hamming_encode_packets.restype = c_int
    L.hamming_packet_channel_generate.argtypes = [u32, c_int, u64, u64, u64, u64, c_int, vp, u64, vp, vp]
    L.hamming_packet_channel_generate.restype = c_int
    L.hamming_coded_bytes.argtypes = [c_int, u64]
    L.hamming_coded_bytes.restype = u64
    L.hamming_data_bytes.argtypes = [c_int, u64]
    L.hamming_data_bytes.restype = u64
    L.hamming_status_string.argtypes = [c_int]
    L.hamming_status_string.restype = ctypes.c_char_p
    L.hamming_last_error.argtypes = []
    L.hamming_last_error.restype = ctypes.c_char_p
    L.hamming_abi_version.restype = c_int
    L.hamming_last_launch_count.restype = c_int
    L.hamming_last_grid_blocks.restype = c_int
    if L.hamming_abi_version() != 1:
        raise RuntimeError("libhamming.so ABI version mismatch")
    _lib = L
    return L


def check(status: int, where: str) -> None:
    if status == 0:
        return
    detail = (lib().hamming_last_error() or b"").decode(errors="replace")
    if status == 6:
        raise HammingError(status, where, detail)
    raise HammingArgumentError(status, where, detail)
