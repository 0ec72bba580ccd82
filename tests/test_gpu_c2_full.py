"""The benchmarked configuration itself (BASELINE.json configs[1], bench.py's C2) checked end to
end against the torch-fp32 oracle (oracle/torch_ref.py, pinned to the reference goldens by
tests/test_torch_ref.py): Llama-3-8B shape (32 layers, d 4096, 32/8 heads, ffn 14336,
vocab 128,256), 8 rank-16 adapters, one 2,048-token prompt prefilled once and hit by the 7
other models through the icarus prefix pool, then batched fused decode -- 32 teacher-forced
steps (all 8 models fed the same tokens, so their caches must stay byte-identical) and 32
free-running steps (each model its own greedy tokens; the oracle follows the GPU's tokens so
every step of the horizon is checked).

The oracle runs on the GPU's own bf16 weights (untiled from the runtime), so the comparison
measures only the kernels' bf16 activations / fp32 accumulation. Tolerance as every GPU
parity test: max |dlogit| <= 3e-2 * max |logit| per step; greedy tokens equal unless the
oracle's top-1 vs the GPU's pick is inside that band (tests/test_acceptance.py:103-108 rule),
ties counted and reported.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
LOGIT_TOL = 3e-2
C2 = dict(num_layers=32, hidden_dim=4096, num_heads=32, num_kv_heads=8, head_dim=128,
          ffn_dim=14336, vocab_size=128256, rope_theta=5e5, rms_eps=1e-5)
N_AD, RANK, ALPHA, PROMPT, TF_STEPS, FREE_STEPS = 8, 16, 32.0, 2048, 32, 32


class Tally:
    def __init__(self):
        self.worst, self.ties, self.checked = 0.0, [], 0

    def check(self, got: np.ndarray, want, gpu_tok: int, label: str) -> None:
        want = want.double().cpu().numpy()
        scale = float(np.abs(want).max())
        err = float(np.abs(got.astype(np.float64) - want).max())
        assert err <= LOGIT_TOL * scale, f"{label}: max|dlogit| {err:.4g} vs scale {scale:.4g}"
        o = int(np.argmax(want))
        assert int(np.argmax(got)) == gpu_tok, f"{label}: emitted token is not the logits' argmax"
        if gpu_tok != o:
            gap = float(want[o] - want[gpu_tok])
            assert gap <= LOGIT_TOL * scale, f"{label}: token {gpu_tok} vs oracle {o}, gap {gap:.4g}"
            self.ties.append((label, o, gpu_tok, round(gap / scale, 5)))
        self.worst = max(self.worst, err / scale)
        self.checked += 1


def test_c2_llama8b_shape_8_adapters_matches_torch_oracle(cuda):
    import torch

    from oracle import torch_ref as R
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig

    cfg = ModelConfig(**C2)
    max_ctx = PROMPT + TF_STEPS + FREE_STEPS + 16
    base = BaseWeights.on_device(cfg, seed=0)
    adapters = [AdapterSet.on_device(cfg, RANK, ALPHA, seed=1 + i, task=f"agent{i}")
                for i in range(N_AD)]
    rt = base.runtime(max_seqs=N_AD + 2, max_context=max_ctx, max_rows=512, adapter_slots=N_AD,
                      lora_rank=RANK, num_pages=PROMPT // 16 + N_AD * 8 + 16)
    pool = KvCachePool(cfg, budget_bytes=8 << 30, mode="icarus")
    prompt = [int(t) for t in np.random.default_rng(1000).integers(1, cfg.vocab_size, PROMPT)]
    sess = [E.new_session(base, a, max_ctx, runtime=rt, capture_logits=True) for a in adapters]
    first = E.prefill(sess[0], prompt, pool=pool, reader="agent0")
    pool.commit(None, prompt, sess[0].cache,
                next_token_fn=lambda p: E.base_next_token_at(sess[0], p), creator="agent0")
    firsts = [first] + [E.prefill(s, prompt, pool=pool, reader=f"agent{i}")
                        for i, s in enumerate(sess[1:], 1)]
    assert firsts == [first] * N_AD  # the stored chunk-end base token (src/engine.py:135-139)
    assert all(s.ledger.prefix_hit_tokens == PROMPT for s in sess[1:])
    assert all(s.cache.pages[:PROMPT // 16] == sess[0].cache.pages[:PROMPT // 16] for s in sess)

    tally = Tally()
    with R.fp32_matmul():
        ref = R.TorchRef(R.Weights.from_device(R.Shape(**C2), rt.dw), max_pos=max_ctx)
        r0 = ref.session(None, capacity=max_ctx)
        r_first = ref.prefill(r0, prompt)
        tally.check(sess[0].last_logits, r0.last_logits, first, "prefill")
        del r_first
        refs = []
        for a in adapters:
            r = ref.session(R.Adapter.from_slots(rt.slots, rt.slots.slot_of(a)), capacity=max_ctx)
            r.copy_prefix(r0, PROMPT)
            refs.append(r)
        del r0
        # teacher-forced: every model consumes the same tokens
        forced = [first] + [int(t) for t in np.random.default_rng(7).integers(1, cfg.vocab_size, TF_STEPS - 1)]
        for step, t in enumerate(forced):
            got = E.decode_step_batch(sess, [t] * N_AD)
            ref.decode_fused(refs, [t] * N_AD)
            for i in range(N_AD):
                tally.check(sess[i].last_logits, refs[i].last_logits, got[i], f"tf step {step} agent{i}")
        fps = {s.cache.fingerprint() for s in sess}
        assert len(fps) == 1, "adapted models wrote different KV bytes"
        n = sess[0].cache.position_count
        for layer in (0, 15, 31):
            k, v = sess[0].cache.rows(layer, 0, n)
            rk = refs[0].k[layer, :n].view(k.shape).cpu().numpy()
            rv = refs[0].v[layer, :n].view(v.shape).cpu().numpy()
            assert np.abs(k - rk).max() <= 2e-2 * np.abs(rk).max() + 1e-2, f"K layer {layer}"
            assert np.abs(v - rv).max() <= 2e-2 * np.abs(rv).max() + 1e-2, f"V layer {layer}"
        # free-running: each model its own greedy tokens; the oracle follows the GPU's tokens
        toks = got
        for step in range(FREE_STEPS):
            nxt = E.decode_step_batch(sess, toks)
            ref.decode_fused(refs, toks)
            for i in range(N_AD):
                tally.check(sess[i].last_logits, refs[i].last_logits, nxt[i], f"free step {step} agent{i}")
            toks = nxt
    print(f"C2 full config: {tally.checked} steps checked, worst relative logit error "
          f"{tally.worst:.3e}, {len(tally.ties)} oracle ties {tally.ties[:8]}")
    for s in sess:
        s.close()
    del ref, refs
    torch.cuda.empty_cache()
