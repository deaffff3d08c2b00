"""Multi-process (world_size 2, gloo, CPU) coverage of the N > 1 path: plan
sharding, max-over-ranks timing, work sums and the result gather used by
bench.py --gpus N (no GPU needed)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2411_03416_b200 import dist as D

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        r, w, lr = D.env_rank()
        assert (r, w, lr) == (rank, world, rank)
        start, stop = D.shard(4097, w, r)
        t = D.reduce_max(10.0 + r)
        n = D.reduce_sum(stop - start)
        D.barrier()
        g = D.gather_summaries({"plan": np.arange(start, stop), "rank": np.full(stop - start, r)})
        out[rank] = (start, stop, t, n, g["plan"].tolist(), g["rank"].tolist())
    finally:
        dist.destroy_process_group()


def test_shard_covers_batch():
    from paper_2411_03416_b200.dist import shard

    for total, world in [(4096, 1), (4096, 8), (4097, 3), (5, 8)]:
        spans = [shard(total, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == total
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) <= 1


@pytest.mark.timeout(120)
def test_two_ranks_gloo():
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    (s0, e0, t0, n0, plans0, ranks0), (s1, e1, t1, n1, plans1, ranks1) = res[0], res[1]
    assert (s0, e0, s1, e1) == (0, 2049, 2049, 4097)
    assert t0 == t1 == 11.0            # max over ranks
    assert n0 == n1 == 4097            # work summed over ranks
    assert plans0 == plans1 == list(range(4097))  # gather in plan order
    assert ranks0[:2049] == [0] * 2049 and ranks0[2049:] == [1] * 2048


@pytest.mark.timeout(300)
def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` without a launcher re-runs itself under
    torch.distributed.run (one rank per device), and its timed region takes
    the max time over ranks and sums the work: driven here on CPU (gloo) with
    the CPU stand-in engine (--stub-engine)."""
    import json
    import subprocess
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--stub-engine",
                          "--steps", "3", "--warmup", "1", "--plans", "64"],
                         capture_output=True, text=True, env=env, timeout=280)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["plans_total"] == 128
    assert line["evals_all"] == 128 * 3 * 999  # every plan of both shards, 3 iterations, F = N - 1
    assert line["value"] == pytest.approx(line["evals_all"] / (line["ms_per_step"] * 3 / 1e3))
    # the world size must match --gpus
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    bad = subprocess.run([sys.executable, os.path.join(repo, "bench.py"), "--gpus", "2", "--stub-engine"],
                         capture_output=True, text=True, env=env, timeout=120)
    assert bad.returncode != 0 and "WORLD_SIZE" in bad.stderr
