"""Multi-process (world size 2, gloo on CPU) coverage of the N>1 path: stream
sharding for config 5 and the result gather bench.py performs after its timed
region (MAX of device time, SUM of frames, gather of checksums)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_1810_03988_b200.shard import RankResult, aggregate_fps, gather_results, shard_streams


def test_shard_streams_partition():
    for n, world in ((64, 1), (64, 2), (64, 4), (64, 8), (10, 3), (3, 4)):
        parts = [shard_streams(n, world, r) for r in range(world)]
        flat = [s for p in parts for s in p]
        assert flat == list(range(n))  # disjoint, contiguous, complete
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
    assert shard_streams(64, 8, 3) == list(range(24, 32))
    with pytest.raises(ValueError):
        shard_streams(64, 2, 2)


def test_gather_single_process():
    ms, frames, sums = gather_results(RankResult(frames=5, device_ms=10.0, checksum=7))
    assert (ms, frames, sums) == (10.0, 5, [7])
    assert aggregate_fps(500, 1000.0) == 500.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = shard_streams(64, world, rank)
        # each rank "stitches" its streams; device time differs per rank
        res = RankResult(frames=len(mine) * 3, device_ms=100.0 + 25.0 * rank, checksum=sum(mine))
        ms, frames, sums = gather_results(res)
        out[rank] = (mine[0], mine[-1], ms, frames, sums, aggregate_fps(frames, ms))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        r0, r1 = out[0], out[1]
    assert (r0[0], r0[1]) == (0, 31) and (r1[0], r1[1]) == (32, 63)
    for r in (r0, r1):
        assert r[2] == 125.0                       # max over ranks
        assert r[3] == 64 * 3                      # all frames
        assert r[4] == [sum(range(32)), sum(range(32, 64))]
        assert abs(r[5] - 64 * 3 / 0.125) < 1e-9   # whole-job frames/s
