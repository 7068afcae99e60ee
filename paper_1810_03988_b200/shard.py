"""Multi-GPU sharding of independent rigs / streams.

The stitching path has no exchange step between independent camera rigs, so
N GPUs run N disjoint shards with no data-path collective (weak scaling when
every rank gets the same share). torch.distributed (NCCL on GPUs, gloo on CPU)
is used only after the timed work: a MAX-reduce of per-rank device time and a
gather of per-rank results (frame counts, panorama checksums), the
"NCCL only to gather results" of the north star.
"""
from dataclasses import dataclass

import torch


def shard_streams(n_streams, world, rank):
    """Contiguous block of stream ids for `rank` (config 5: 64 streams over
    1/2/4/8 GPUs -> 64/8/16/32 per rank; remainders go to the low ranks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_streams, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return list(range(lo, hi))


@dataclass
class RankResult:
    frames: int
    device_ms: float
    checksum: int


def gather_results(res: RankResult, device=None):
    """All ranks contribute; returns (max device ms, total frames, checksums by rank).
    Works for world size 1 without an initialised process group."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return res.device_ms, res.frames, [res.checksum]
    dev = device if device is not None else torch.device("cpu")
    t = torch.tensor([res.device_ms], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    f = torch.tensor([res.frames], dtype=torch.int64, device=dev)
    dist.all_reduce(f, op=dist.ReduceOp.SUM)
    c = torch.tensor([res.checksum], dtype=torch.int64, device=dev)
    allc = [torch.zeros_like(c) for _ in range(dist.get_world_size())]
    dist.all_gather(allc, c)
    return float(t.item()), int(f.item()), [int(x.item()) for x in allc]


def aggregate_fps(total_frames, max_device_ms):
    """Whole-job throughput: frames of all ranks over the slowest rank's time."""
    return total_frames / (max_device_ms / 1e3) if max_device_ms > 0 else 0.0


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_argv(script, argv, nproc, python=None, port=None):
    """Command line that re-launches `script argv` as `nproc` ranks on this
    node (one process per GPU), the way the driver launches multi-GPU runs:
    torch.distributed.run, rendezvous on 127.0.0.1."""
    import sys
    return [python or sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
            f"--nproc-per-node={int(nproc)}", "--master-addr=127.0.0.1",
            f"--master-port={int(port or free_port())}", script, *argv]


def maybe_self_launch(script, argv, nproc, env=None):
    """bench.py --gpus N run without torchrun: spawn the N ranks here and
    return their exit code; None when already inside a launched job (or N=1)."""
    import os
    import subprocess
    env = os.environ if env is None else env
    if nproc <= 1 or "WORLD_SIZE" in env:
        return None
    return subprocess.call(torchrun_argv(script, argv, nproc), env=dict(env))
