"""Data-parallel request sharding on >= 2 GPUs (BASELINE.json configs[4]):
one process per GPU over NCCL, requests routed by prefix affinity (dist.route), every rank a
full replica with its own page arena and prefix pool -- no collective on the hot path. The
union of the ranks' outputs must equal one GPU serving every request, bitwise, and the
timing / P95 collectives must work over NCCL. Skips on a box with fewer than two GPUs (the
same logic runs over gloo on CPU in tests/test_dist.py)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
C1 = dict(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128, ffn_dim=1024,
          vocab_size=1024)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _serve(prompts, max_new):
    from oracle import icarus_oracle as O
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200 import model as M
    shape = O.Shape(**C1)
    w = O.bf16_weights(O.init_base(shape, 0))
    cfg = M.ModelConfig(**C1)
    base = M.BaseWeights(cfg, w["embed"], [dict(l) for l in w["layers"]], w["final_gain"], w["lm_head"])
    ads = [M.AdapterSet(cfg, a["rank"], a["alpha"], M.DECODER_TARGETS,
                        [{t: M.LowRankPair(M.Param(p["a"]), M.Param(p["b"])) for t, p in per.items()}
                         for per in a["layers"]])
           for a in (O.bf16_adapter(x) for x in O.make_agents(shape, 2, seed=1))]
    rt = base.runtime(max_seqs=16, max_context=256, max_rows=128, adapter_slots=2, lora_rank=8)
    out = {}
    sessions = [E.new_session(base, ads[i % 2], 128, runtime=rt) for i, _ in prompts]
    res = E.generate_batch(sessions, [p for _, p in prompts], max_new)
    for (i, _), toks in zip(prompts, res):
        out[i] = toks
    for s in sessions:
        s.close()
    return out


def _worker(rank, world, port, prompts, max_new, q):
    import torch
    import torch.distributed as dist
    from paper_2603_13281_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    mine = D.shard(list(enumerate(prompts)), world, rank, prompts=prompts)
    got = _serve(mine, max_new)
    parts = [None] * world
    dist.all_gather_object(parts, got)
    slowest = D.max_over_ranks(float(rank + 1), device="cuda")
    p95 = D.global_p95([float(rank * 10 + k) for k in range(10)])
    if rank == 0:
        merged = {}
        for p in parts:
            merged.update(p)
        q.put((merged, [len(p) for p in parts], slowest, p95))
    dist.barrier()
    dist.destroy_process_group()


def test_two_gpu_sharded_serving_equals_one_gpu(cuda):
    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs at least 2 GPUs")
    rng = np.random.default_rng(5)
    shared = [int(t) for t in rng.integers(1, 1024, 32)]
    prompts = [shared + [int(t) for t in rng.integers(1, 1024, int(rng.integers(3, 20)))] for _ in range(8)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, prompts, 6, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, counts, slowest, p95 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(merged) == list(range(8)) and sum(counts) == 8 and min(counts) > 0
    alone = _serve(list(enumerate(prompts)), 6)
    assert merged == alone
    assert slowest == 2.0
    from paper_2603_13281_b200.dist import p95_nearest_rank
    assert p95 == p95_nearest_rank([float(r * 10 + k) for r in range(2) for k in range(10)])
