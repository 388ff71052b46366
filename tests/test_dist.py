"""Multi-process (gloo, world_size 2, CPU) coverage of the sharding /
max-over-ranks / verification-gather logic used by bench.py --gpus N - both
through paper_2507_11978_b200.dist directly and through bench.py's own
self-spawn + shard + verify path (``--cpu-check``: the oracle stands in for
the kernels, gloo for NCCL)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2507_11978_b200.dist import shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 4096, 4097):
        for w in (1, 2, 3, 8):
            got = [shard_range(total, r, w) for r in range(w)]
            assert got[0][0] == 0 and got[-1][1] == total
            for (a, b), (c, d) in zip(got, got[1:]):
                assert b == c
            sizes = [b - a for a, b in got]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    import oracle
    from paper_2507_11978_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    x = rng.uniform(-1, 1, (64, 32)).astype(np.float32)       # same global problem
    lo, hi = D.shard_range(64, rank, world)
    mine = oracle.softmax(x[lo:hi])                             # this rank's shard
    err = float(np.abs(mine - oracle.softmax(x)[lo:hi]).max())
    t = D.max_over_ranks(float(rank + 1))
    errs = D.gather_scalars(err)
    out.put((rank, t, errs, (lo, hi)))
    dist.destroy_process_group()


def test_two_rank_gloo_shard_and_verify():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [2.0, 2.0]            # max over ranks
    assert res[0][2] == res[1][2] and len(res[0][2]) == 2
    assert max(res[0][2]) == 0.0
    assert res[0][3] == (0, 32) and res[1][3] == (32, 64)


ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("world", [2, 3])
def test_bench_gpus_n_self_spawns_and_shards(world):
    """`bench.py --gpus N` re-executes under torch.distributed.run, each rank
    builds its row shard of ONE global problem, the timing is the max over
    ranks, and one gather of per-rank errors verifies every shard."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", str(world),
                          "--cpu-check", "--steps", "3", "--warmup", "3", "--cpu-rows", "100"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["impl"] == "cpu-check" and line["n_gpus"] == world
    assert line["shard_starts"] == [float(shard_range(100, r, world)[0]) for r in range(world)]
    assert line["verify"]["ok"] and len(line["verify"]["max_err_over_tol_per_rank"]) == world
    assert line["value"] > 0 and line["scaling"] == "strong"
