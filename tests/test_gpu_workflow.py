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
