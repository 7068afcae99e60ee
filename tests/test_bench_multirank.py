"""bench.py --gpus 2 end to end: the bench launches its two ranks itself
(torch.distributed.run on 127.0.0.1), each rank runs its own rig, and rank 0
prints one JSON line for the whole job. On the single GPU of a test box both
ranks share cuda:0 (LPB_RANKS_ON_ONE_GPU=1) and talk over gloo; the driver's
8-GPU run uses one GPU per rank over NCCL with the same code."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["cfg1", "cfg5"])
def test_bench_two_ranks(config):
    env = dict(os.environ, LPB_RANKS_ON_ONE_GPU="1", LPB_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config,
                        "--steps", "6", "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--no-profile",
                        "--no-parity"], capture_output=True, text=True, env=env, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["value"] > 0
    cs = line["rank_checksums"]
    assert len(cs) == 2
    if config == "cfg1":  # each rank stitches its own seeded frames
        assert cs[0] != cs[1]
