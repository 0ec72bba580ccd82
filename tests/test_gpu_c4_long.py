"""BASELINE.json configs[3] (C4, long-context shared KV) checked end to end against the
torch-fp32 oracle (oracle/torch_ref.py, pinned to the reference goldens by
tests/test_torch_ref.py): Llama-3-8B shape, 8 rank-16 adapters on ONE 32,768-token prompt,
prefilled once (64 prefill forwards of 512 rows) and hit by the 7 other models through the
icarus prefix pool, then batched fused decode at 32k context -- the configuration whose
attention runs the long-chunk path (128-page work items, 16-lane softmax form, in-kernel
merge of 17 chunk partials per row).

All 8 models run on the GPU; the oracle follows two of them (the first and the last adapter
slot) -- a 32k fp32 K/V cache is 8.6 GB per oracle session. 4 teacher-forced steps (all 8
models fed the same tokens, so the 8 caches must stay byte-identical) and 4 free-running
steps (each model its own greedy tokens; the oracle follows the GPU's tokens). Tolerance as
tests/test_gpu_c2_full.py: max |dlogit| <= 3e-2 * max |logit| per step; greedy tokens equal
unless the oracle's top-2 gap is inside that band (tests/test_acceptance.py:103-108 rule).
The oracle prefills in 2,048-token chunks (its attention materialises the score matrix).
"""

import numpy as np
import pytest

from test_gpu_c2_full import C2, LOGIT_TOL, Tally  # noqa: F401  (same model, same rule)

pytestmark = pytest.mark.gpu
N_AD, RANK, ALPHA, PROMPT, TF_STEPS, FREE_STEPS = 8, 16, 32.0, 32768, 4, 4
FOLLOW = (0, 7)


def test_c4_32k_shared_prompt_8_adapters_matches_torch_oracle(cuda):
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
                      lora_rank=RANK, num_pages=PROMPT // 16 + N_AD * 4 + 16)
    assert rt.chunk_pages == 128  # the long-chunk attention path under test
    pool = KvCachePool(cfg, budget_bytes=64 << 30, mode="icarus")
    prompt = [int(t) for t in np.random.default_rng(4000).integers(1, cfg.vocab_size, PROMPT)]
    sess = [E.new_session(base, a, max_ctx, runtime=rt, capture_logits=True) for a in adapters]
    first = E.prefill(sess[0], prompt, pool=pool, reader="agent0")
    pool.commit(None, prompt, sess[0].cache,
                next_token_fn=lambda p: E.base_next_token_at(sess[0], p), creator="agent0")
    firsts = [first] + [E.prefill(s, prompt, pool=pool, reader=f"agent{i}")
                        for i, s in enumerate(sess[1:], 1)]
    assert firsts == [first] * N_AD
    assert all(s.ledger.prefix_hit_tokens == PROMPT for s in sess[1:])
    assert all(s.cache.pages[:PROMPT // 16] == sess[0].cache.pages[:PROMPT // 16] for s in sess)

    tally = Tally()
    with R.fp32_matmul():
        ref = R.TorchRef(R.Weights.from_device(R.Shape(**C2), rt.dw), max_pos=max_ctx)
        r0 = ref.session(None, capacity=max_ctx)
        for c0 in range(0, PROMPT, 2048):
            ref.prefill(r0, prompt[c0:c0 + 2048])
        tally.check(sess[0].last_logits, r0.last_logits, first, "prefill")
        refs = []
        for i in FOLLOW:
            r = ref.session(R.Adapter.from_slots(rt.slots, rt.slots.slot_of(adapters[i])),
                            capacity=max_ctx)
            r.copy_prefix(r0, PROMPT)
            refs.append(r)
        del r0
        torch.cuda.empty_cache()
        forced = [first] + [int(t) for t in
                            np.random.default_rng(9).integers(1, cfg.vocab_size, TF_STEPS - 1)]
        for step, t in enumerate(forced):
            got = E.decode_step_batch(sess, [t] * N_AD)
            ref.decode_fused(refs, [t] * len(FOLLOW))
            for j, i in enumerate(FOLLOW):
                tally.check(sess[i].last_logits, refs[j].last_logits, got[i], f"tf step {step} agent{i}")
        # the prefix pages are the same page ids (asserted above); the decode steps' K/V live in
        # each session's private tail page -- byte-identical across the 8 models
        n = sess[0].cache.position_count
        for layer in range(cfg.num_layers):
            tails = {s.cache.arena.read_raw(layer, s.cache.pages, PROMPT, n) for s in sess}
            assert len(tails) == 1 and len(next(iter(tails))[0]) > 0, \
                f"adapted models wrote different KV bytes (layer {layer})"
        toks = got
        for step in range(FREE_STEPS):
            nxt = E.decode_step_batch(sess, toks)
            ref.decode_fused(refs, [toks[i] for i in FOLLOW])
            for j, i in enumerate(FOLLOW):
                tally.check(sess[i].last_logits, refs[j].last_logits, nxt[i], f"free step {step} agent{i}")
            toks = nxt
    print(f"C4 32k: {tally.checked} steps checked, worst relative logit error {tally.worst:.3e}, "
          f"{len(tally.ties)} oracle ties {tally.ties[:8]}")
    for s in sess:
        s.close()
    del ref, refs
    torch.cuda.empty_cache()


def test_c3_shaped_shared_8k_prefix_wide_batches_match_torch_oracle(cuda):
    """BASELINE.json configs[2] (C3) in miniature, end to end against the torch-fp32 oracle:
    one 8,192-token prefix shared by 16 sessions over 8 adapters (64-page attention items:
    the long-chunk path with 129 query entries per item), their distinct suffixes prefilled
    in ONE shared forward (engine.prefill_batch), wide fused decode steps (32 and 40 rows),
    and 4 new sessions whose prefill rides in a decode step (engine.step_batch). The oracle
    follows one session of the first wave and one piggybacked session through every step."""
    import torch

    from oracle import torch_ref as R
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig

    cfg = ModelConfig(**C2)
    prefix_len, max_ctx = 8192, 8192 + 256
    base = BaseWeights.on_device(cfg, seed=0)
    adapters = [AdapterSet.on_device(cfg, RANK, ALPHA, seed=1 + i, task=f"agent{i}")
                for i in range(N_AD)]
    rt = base.runtime(max_seqs=24, max_context=max_ctx, max_rows=512, adapter_slots=N_AD,
                      lora_rank=RANK, num_pages=prefix_len // 16 + 24 * 12 + 16)
    assert rt.chunk_pages == 64
    rng = np.random.default_rng(33)
    prefix = [int(t) for t in rng.integers(1, cfg.vocab_size, prefix_len)]
    pool = KvCachePool(cfg, budget_bytes=64 << 30, mode="icarus")
    writer = E.new_session(base, None, max_ctx, runtime=rt)
    E.prefill(writer, prefix, pool=pool)
    pool.commit(None, prefix, writer.cache, next_token_fn=lambda p: E.base_next_token_at(writer, p))
    writer.close()
    wave1 = [E.new_session(base, adapters[i % N_AD], max_ctx, runtime=rt, capture_logits=True)
             for i in range(16)]
    suffix1 = [[int(t) for t in rng.integers(1, cfg.vocab_size, int(rng.integers(10, 80)))] for _ in wave1]
    toks = E.prefill_batch(wave1, [prefix + s for s in suffix1], pool=pool)
    assert all(s.ledger.prefix_hit_tokens == prefix_len for s in wave1)
    A, B = 3, 1  # followed: wave-1 session 3, piggybacked session 1

    tally = Tally()
    with R.fp32_matmul():
        ref = R.TorchRef(R.Weights.from_device(R.Shape(**C2), rt.dw), max_pos=max_ctx)
        r0 = ref.session(None, capacity=max_ctx)
        for c0 in range(0, prefix_len, 2048):
            ref.prefill(r0, prefix[c0:c0 + 2048])

        def follow(sess, suffix):
            r = ref.session(R.Adapter.from_slots(rt.slots, rt.slots.slot_of(sess.adapter)), capacity=max_ctx)
            r.copy_prefix(r0, prefix_len)
            ref.prefill(r, suffix)
            return r

        ra = follow(wave1[A], suffix1[A])
        tally.check(wave1[A].last_logits, ra.last_logits, toks[A], "wave1 prefill")
        for step in range(3):  # 32-row fused steps
            nxt = E.decode_step_batch(wave1, toks)
            ref.decode_fused([ra], [toks[A]])
            tally.check(wave1[A].last_logits, ra.last_logits, nxt[A], f"wave1 step {step}")
            toks = nxt
        wave2 = [E.new_session(base, adapters[(5 + i) % N_AD], max_ctx, runtime=rt, capture_logits=True)
                 for i in range(4)]
        suffix2 = [[int(t) for t in rng.integers(1, cfg.vocab_size, int(rng.integers(10, 80)))] for _ in wave2]
        nxt, toks2 = E.step_batch(wave1, toks, wave2, [prefix + s for s in suffix2], pool=pool)
        ref.decode_fused([ra], [toks[A]])
        tally.check(wave1[A].last_logits, ra.last_logits, nxt[A], "fused step (decode + piggybacked prefill)")
        rb = follow(wave2[B], suffix2[B])
        tally.check(wave2[B].last_logits, rb.last_logits, toks2[B], "piggybacked prefill")
        everyone, toks = wave1 + wave2, nxt + toks2
        for step in range(2):  # 40-row fused steps
            nxt = E.decode_step_batch(everyone, toks)
            ref.decode_fused([ra, rb], [toks[A], toks[16 + B]])
            tally.check(everyone[A].last_logits, ra.last_logits, nxt[A], f"all step {step} A")
            tally.check(everyone[16 + B].last_logits, rb.last_logits, nxt[16 + B], f"all step {step} B")
            toks = nxt
    print(f"C3-shaped: {tally.checked} checks, worst relative logit error {tally.worst:.3e}, "
          f"{len(tally.ties)} oracle ties {tally.ties[:8]}")
    for s in everyone:
        s.close()
    del ref, r0, ra, rb
    torch.cuda.empty_cache()
