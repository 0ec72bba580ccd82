"""Multi-rank host logic on CPU (gloo, world size 2): routing, max-over-ranks timing and the
global nearest-rank P95. The hot path itself has no collective (replicas only)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_13281_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = D.max_over_ranks(1.5 + rank)
        lat = [float(rank * 100 + i) for i in range(20)]
        p95 = D.global_p95(lat)
        prompts = [[7] * 32] * 6 + [[9] * 32] * 2
        mine = D.shard(list(range(8)), world, rank, prompts)
        total = D.sum_over_ranks(float(len(mine)))        # whole-job token / step totals (C5)
        q.put((rank, t, p95, mine, total))
    finally:
        dist.destroy_process_group()


def test_two_rank_timing_and_p95_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_lat = [float(r * 100 + i) for r in range(2) for i in range(20)]
    for rank, t, p95, mine, total in res:
        assert t == 2.5                                   # max over ranks
        assert total == 8.0                               # sum over ranks
        assert p95 == D.p95_nearest_rank(all_lat) == 117.0  # rank ceil(0.95*40)=38
    shards = [set(m) for _, _, _, m, _ in res]
    assert shards[0].isdisjoint(shards[1]) and shards[0] | shards[1] == set(range(8))
    assert len(shards[0]) == len(shards[1]) == 4       # weak scaling: equal per-GPU work


def test_route_balances_and_keeps_prefix_affinity():
    rng = np.random.default_rng(0)
    a = [int(t) for t in rng.integers(1, 100, 48)]
    b = [int(t) for t in rng.integers(1, 100, 48)]
    prompts = [a] * 8 + [b] * 8
    ranks = D.route(prompts, 4)
    assert sorted(np.bincount(ranks, minlength=4)) == [4, 4, 4, 4]
    # with balance satisfied, each prefix touches as few GPUs as possible (2 of 4)
    assert len(set(ranks[:8])) == 2 and len(set(ranks[8:])) == 2
    assert D.route(prompts, 1) == [0] * 16


def test_p95_nearest_rank_matches_reference_definition():
    assert D.p95_nearest_rank([]) == 0.0
    assert D.p95_nearest_rank([3.0]) == 3.0
    xs = list(range(1, 101))
    assert D.p95_nearest_rank(xs) == 95
    assert D.p95_nearest_rank(list(reversed(xs))) == 95


def test_prefix_key_uses_first_block_chain_hash():
    from paper_2603_13281_b200.kvpool import chain_hash
    toks = list(range(40))
    assert D.prefix_key(toks) == chain_hash(0, tuple(range(16)))
    assert D.prefix_key(toks[:10]) == 0


def test_bench_gpus_flag_relaunches_one_rank_per_gpu(monkeypatch):
    """`bench.py --gpus N` without a torchrun environment re-launches itself under
    torch.distributed.run with N processes on 127.0.0.1 (--gpus was ignored)."""
    import subprocess
    import sys

    import bench
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(subprocess, "call", fake_call)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "8"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "8"]
    # under torchrun a disagreeing --gpus is an error, not a silent single rank
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit) as ex2:
        bench.main()
    assert "disagrees" in str(ex2.value.code)
