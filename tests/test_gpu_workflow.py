"""Continuous-batching multi-agent serving (paper_2603_13281_b200.workflow, C3 semantics) on a
C1-shaped model: every request completes, later turns and other models reuse the shared prefix
through the pool, and every turn's tokens equal the tokens of the same turn decoded alone
(batch invariance of the fused multi-model step)."""

import numpy as np
import pytest

from oracle import icarus_oracle as O

pytestmark = pytest.mark.gpu

C1 = dict(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128, ffn_dim=1024,
          vocab_size=1024)


def test_workflow_batched_equals_alone(cuda):
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200 import workflow as W
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, LowRankPair, ModelConfig, Param
    shape = O.Shape(**C1)
    w = O.bf16_weights(O.init_base(shape, 0))
    cfg = ModelConfig(**C1)
    base = BaseWeights(cfg, w["embed"], [dict(l) for l in w["layers"]], w["final_gain"], w["lm_head"])
    ads = []
    for i, a in enumerate(O.make_agents(shape, 3, seed=1)):
        a = O.bf16_adapter(a)
        ads.append(AdapterSet(cfg, a["rank"], a["alpha"], ("q", "o", "gate", "up", "down"),
                              [{t: LowRankPair(Param(p["a"]), Param(p["b"])) for t, p in per.items()}
                               for per in a["layers"]], f"agent{i}"))
    wcfg = W.WorkflowConfig(requests=6, num_agents=3, prefix_len=64, question_min=8, question_max=16,
                            turns_min=2, turns_max=3, output_min=4, output_max=8, obs_min=4, obs_max=8,
                            seed=3, max_batch=4)
    prefix, reqs = W.make_workload(wcfg, cfg.vocab_size)
    max_ctx = (W.max_context_tokens(prefix, reqs) + 31) // 16 * 16
    rt = base.runtime(max_seqs=12, max_context=max_ctx, max_rows=64, adapter_slots=3, lora_rank=8,
                      num_pages=256)
    pool = KvCachePool(cfg, budget_bytes=256 << 20, mode="icarus")
    assert W.warm_prefix(base, pool, prefix, max_ctx, runtime=rt) == 64
    rep = W.serve(base, ads, pool, prefix, reqs, wcfg, max_ctx, runtime=rt)
    assert rep.completed == len(reqs)
    assert rep.turns == sum(len(r.turns) for r in reqs)
    assert rep.max_live == wcfg.max_batch
    assert rep.prefix_hit_tokens >= len(reqs) * 64       # every first turn hits the prefix
    assert rep.cross_model_hit_tokens > 0                  # later turns reuse other models' KV
    assert rep.p95_latency_ms > 0 and rep.decode_tok_s > 0
    # each turn alone (fresh session, no pool), teacher-forced on the same context
    for r in reqs:
        ctx = list(prefix)
        for j, t in enumerate(r.turns):
            ctx = ctx + list(t.new_tokens)
            s = E.new_session(base, ads[t.agent], max_ctx, runtime=rt)
            alone = E.generate(s, ctx, t.output_len)
            s.close()
            assert alone == rep.outputs[(r.rid, j)], (r.rid, j)
            ctx = ctx + alone


@pytest.mark.parametrize("mode", ["icarus", "baseline"])
def test_workflow_counters_equal_reference_simulate_run(cuda, mode):
    """The reference's serving loop (simulate.run, src/simulate.py:254-364) on the same trace
    (tests/golden/workflow_c1.json, produced by the unmodified reference): token conservation,
    prefill / prefix-hit / cross-model tokens, decode steps, ledger KV bytes, peak pool bytes and
    evictions are determined by the trace's lengths and the pool rules, so the continuous-
    batching driver must reproduce them exactly in both pool modes."""
    import json
    from pathlib import Path

    from paper_2603_13281_b200 import workflow as W
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.metrics import Ledger
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, LowRankPair, ModelConfig, Param
    from paper_2603_13281_b200.runtime import Runtime
    g = json.loads((Path(__file__).resolve().parent / "golden" / "workflow_c1.json").read_text())
    want = g["reports"][mode]
    shape = O.Shape(**C1)
    w = O.bf16_weights(O.init_base(shape, 0))
    cfg = ModelConfig(**C1)
    base = BaseWeights(cfg, w["embed"], [dict(l) for l in w["layers"]], w["final_gain"], w["lm_head"])
    ads = []
    for i, a in enumerate(O.make_agents(shape, 4, seed=1)):
        a = O.bf16_adapter(a)
        ads.append(AdapterSet(cfg, a["rank"], a["alpha"], ("q", "o", "gate", "up", "down"),
                              [{t: LowRankPair(Param(p["a"]), Param(p["b"])) for t, p in per.items()}
                               for per in a["layers"]], f"agent{i}"))
    reqs = [W.Request(rid, tuple(W.Turn(a, tuple(toks), out) for a, toks, out in turns))
            for rid, turns in enumerate(g["trace"])]
    wcfg = W.WorkflowConfig(requests=len(reqs), num_agents=4, prefix_len=0, max_batch=4)
    rt = Runtime(base, max_seqs=16, max_context=256, max_rows=128, adapter_slots=4, lora_rank=8,
                 num_pages=512)
    pool = KvCachePool(cfg, budget_bytes=g["budget_bytes"], mode=mode)
    ledger = Ledger()
    rep = W.serve(base, ads, pool, (), reqs, wcfg, 256, runtime=rt, ledger=ledger)
    st, led = pool.stats(), ledger.snapshot()
    got = {"completed": rep.completed, "eviction_count": st["evicted_blocks"],
           "recompute_tokens": st["recompute_tokens"],
           "swap_bytes": st["swap_out_bytes"] + st["swap_in_bytes"], "peak_kv_bytes": st["peak_bytes"],
           "cross_model_hit_tokens": st["cross_model_hit_tokens"], "prefill_tokens": led["prefill_tokens"],
           "prefix_hit_tokens": led["prefix_hit_tokens"], "decode_steps": led["decode_steps"],
           "param_passes": led["param_passes"], "kv_bytes_read": led["kv_bytes_read"],
           "kv_bytes_written": led["kv_bytes_written"]}
    assert got == {k: want[k] for k in got}
    # token conservation (pkg/tests/test_simulate.py:122-135)
    conserved = 0
    for r in reqs:
        ctx = 0
        for t in r.turns:
            ctx += len(t.new_tokens)
            conserved += ctx
            ctx += t.output_len
    assert led["prefill_tokens"] + led["prefix_hit_tokens"] == conserved
