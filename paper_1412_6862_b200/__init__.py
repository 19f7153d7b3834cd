"""B200-native batched Hamming decoder (arXiv 1412.6862, Islam, Kim & Kim).

The product is the C-ABI library ``libhamming.so`` (include/hamming.h) built
from ``csrc/hamming.cu`` for sm_100a; this package is its thin Python binding
(torch for device memory, streams and process groups only).
"""
from .api import (SecdedResult, channel_generate_secded, decode_secded, encode_secded, secded_coded_bytes)
from .api import (DecodeResult, PacketDecodeResult, TILE, decode_packets, encode_packets, packet_channel_generate,
                  packet_coded_bytes, packet_layout, packet_stride, packet_launch_shape, channel_generate, channel_thresholds, code_nk, coded_bytes, data_bytes,
                  decode, decode_host, encode, hamming_channel_generate, hamming_decode, hamming_decode_host,
                  hamming_encode, host_workspace_bytes, last_grid_blocks, last_launch_count)
from .dist import decode_sharded, shard_range

__all__ = [
    "DecodeResult", "TILE", "channel_generate", "channel_thresholds", "code_nk", "coded_bytes", "data_bytes",
    "decode", "decode_host", "encode", "hamming_channel_generate", "hamming_decode", "hamming_decode_host",
    "hamming_encode", "host_workspace_bytes", "last_grid_blocks", "last_launch_count", "decode_sharded",
    "shard_range", "PacketDecodeResult", "decode_packets", "encode_packets", "packet_channel_generate",
    "packet_coded_bytes", "packet_layout", "packet_stride", "packet_launch_shape", "SecdedResult", "channel_generate_secded",
    "decode_secded", "encode_secded", "secded_coded_bytes",
]
