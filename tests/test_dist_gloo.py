"""Multi-rank host logic on CPU (-m "not gpu"): codeword-range sharding and
the count all_reduce, world size 2 over gloo.  The per-rank decode is the CPU
oracle standing in for the device decode (test-only): the point is that the
shards tile the packet, start on byte/vector boundaries, and that
rank-order concatenation of the shard outputs plus the reduced count equal
the single-rank result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1412_6862_b200.dist import allreduce_count, shard_range


@pytest.mark.parametrize("N", [0, 1, 1023, 1024, 5000, 10 ** 6 + 17, (1 << 39) // 63])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_tiles_and_aligns(N, world):
    prev = 0
    for r in range(world):
        a, b = shard_range(N, r, world)
        assert a == prev and a <= b and a % 1024 == 0
        for m in (3, 6):
            n, k = 2 ** m - 1, 2 ** m - 1 - m
            assert (a * n) % 128 == 0 and (a * k) % 128 == 0  # 16-byte aligned byte offsets
        prev = b
    assert prev == N
    sizes = [shard_range(N, r, world)[1] - shard_range(N, r, world)[0] for r in range(world)]
    if N >= 1024 * world:
        assert max(sizes) - min(sizes) <= 2048


def test_shard_range_rejects_bad_args():
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)
    with pytest.raises(ValueError):
        shard_range(10, 0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, m, N, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    a, b = shard_range(N, rank, world)
    rx, _, _ = oracle.generate(m, 0xD15, a, b - a, p=0.3, q2=0.3)
    data, syn, cnt = oracle.decode(m, rx, b - a)
    count = torch.tensor([cnt], dtype=torch.int64)
    allreduce_count(count)
    np.save(os.path.join(outdir, f"data{rank}.npy"), data)
    np.save(os.path.join(outdir, f"syn{rank}.npy"), syn)
    np.save(os.path.join(outdir, f"cnt{rank}.npy"), count.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("m", [3, 6])
def test_two_rank_gloo_shards_concatenate_to_single_rank(oracle, tmp_path, m):
    world, N = 2, 5 * 1024 + 333
    mp.spawn(_worker, args=(world, _free_port(), m, N, str(tmp_path)), nprocs=world, join=True)
    rx, _, _ = oracle.generate(m, 0xD15, 0, N, p=0.3, q2=0.3)
    wd, ws, wc = oracle.decode(m, rx, N)
    data = np.concatenate([np.load(tmp_path / f"data{r}.npy") for r in range(world)])
    syn = np.concatenate([np.load(tmp_path / f"syn{r}.npy") for r in range(world)])
    assert np.array_equal(data, wd) and np.array_equal(syn, ws)
    for r in range(world):
        assert int(np.load(tmp_path / f"cnt{r}.npy")[0]) == wc
