"""Multi-GPU sharding: codewords are independent (the paper
decodes segments in parallel), so rank r of R owns the contiguous
codeword range [c_r, c_{r+1}) with c_r a multiple of the 1024-codeword tile
(byte offsets c_r*n/8, c_r*k/8 and c_r are then 16-byte aligned; no bit
stitching between ranks).  The only collective is one all_reduce (SUM) of the
8-byte corrected count, stream-ordered after the decode.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .api import TILE, DecodeResult, hamming_decode


def shard_range(n_codewords: int, rank: int, world: int, align: int = TILE) -> tuple[int, int]:
    """[start, end) of rank's shard: floor(r N / R / align) * align; the last
    rank takes the remainder.  Every rank's start is a multiple of `align`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if align < 1:
        raise ValueError("align must be >= 1")

    def edge(r: int) -> int:
        if r >= world:
            return n_codewords
        return (n_codewords * r // world) // align * align

    return edge(rank), edge(rank + 1)


def allreduce_count(count: torch.Tensor, group=None) -> torch.Tensor:
    """Global corrected count: one SUM all_reduce of the int64 [1] tensor."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(count, op=dist.ReduceOp.SUM, group=group)
    return count


def decode_sharded(m: int, rx_local: torch.Tensor, n_local: int, group=None, **kw) -> DecodeResult:
    """Decode this rank's shard, then all-reduce the corrected count, so the
    returned `corrected` is the GLOBAL count while data/syndromes stay local."""
    res = hamming_decode(m, rx_local, n_local, **kw)
    allreduce_count(res.corrected, group)
    return res
