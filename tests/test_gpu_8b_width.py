"""One Llama-3-8B-width layer (BASELINE.json configs[1] shapes: d 4096, 32/8 heads of 128,
ffn 14336, rank-16 adapters) through the batched fused decode step, against the CPU oracle on
the same bf16-representable weights: pins the kernels at the widths the bench runs (GEMM
tilings, stream-K splits, LoRA segments of 2 adapters in one launch, GQA 4:1) rather than
only at C1's d = 256. One layer and a 2048-token vocabulary keep the oracle to ~1 minute.

Tolerance as tests/test_gpu_engine.py: max |dlogit| <= 3e-2 * max |logit| per step, greedy
tokens equal unless the oracle's own top-2 gap is inside that band.
"""

import numpy as np
import pytest

from oracle import icarus_oracle as O

pytestmark = pytest.mark.gpu
LOGIT_TOL = 3e-2
C8 = dict(num_layers=1, hidden_dim=4096, num_heads=32, num_kv_heads=8, head_dim=128, ffn_dim=14336,
          vocab_size=2048, rope_theta=500000.0, rms_eps=1e-5)


def _check(got, want, label):
    scale = float(np.abs(want).max())
    err = float(np.abs(got - want).max())
    assert err <= LOGIT_TOL * scale, f"{label}: max|dlogit| {err:.4g} vs scale {scale:.4g}"
    g, o = int(np.argmax(got)), int(np.argmax(want))
    if g != o:
        assert float(want[o] - want[g]) <= LOGIT_TOL * scale, f"{label}: argmax {g} vs {o}"
    return err / scale


def test_llama8b_width_layer_batched_decode_matches_oracle(cuda):
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200 import model as M
    shape = O.Shape(**C8)
    w = O.bf16_weights(O.init_base(shape, 0))
    ads = [O.bf16_adapter(a) for a in O.make_agents(shape, 2, seed=1, rank=16, alpha=32.0)]
    cfg = M.ModelConfig(**C8)
    base = M.BaseWeights(cfg, w["embed"], [dict(lw) for lw in w["layers"]], w["final_gain"], w["lm_head"])
    agents = [M.AdapterSet(cfg, ad["rank"], ad["alpha"], M.DECODER_TARGETS,
                           [{t: M.LowRankPair(M.Param(p["a"]), M.Param(p["b"])) for t, p in per.items()}
                            for per in ad["layers"]], f"agent{i}")
              for i, ad in enumerate(ads)]
    rt = base.runtime(max_seqs=4, max_context=64, max_rows=16, adapter_slots=2, lora_rank=16)
    prompt = [int(t) for t in np.random.default_rng(3).integers(1, 2048, 4)]
    # oracle: one base prefill, then one session per agent over copies of its cache
    ref0 = O.Session(shape, w, None)
    first = ref0.prefill(prompt)
    refs = [O.Session(shape, w, ad, k=[x.copy() for x in ref0.k], v=[x.copy() for x in ref0.v])
            for ad in ads]
    sess = [E.new_session(base, a, 64, runtime=rt, capture_logits=True) for a in agents]
    assert [E.prefill(s, prompt) for s in sess] == [first, first]
    _check(sess[0].last_logits, ref0.last_logits, "prefill")
    toks = [first, first]
    worst = 0.0
    oracle_toks, oracle_logits = [], []
    for step in range(2):
        E.decode_step_batch(sess, toks)
        toks = [r.decode_fused(t) for r, t in zip(refs, toks)]  # teacher-forced on the oracle
        oracle_toks.append(list(toks))
        oracle_logits.append([r.last_logits.copy() for r in refs])
        for i, (s, r) in enumerate(zip(sess, refs)):
            worst = max(worst, _check(s.last_logits, r.last_logits, f"agent{i} step {step}"))
    # pin the torch-fp32 oracle (the full-depth checker of tests/test_gpu_c2_full.py) to the
    # bitwise oracle at this width: same weights, prefill + the same two teacher-forced steps
    import torch
    from oracle import torch_ref as R
    with R.fp32_matmul():
        tr = R.TorchRef(R.Weights.from_oracle(R.Shape(**C8), w, device="cuda"), max_pos=64)
        t0 = tr.session(None)
        assert tr.prefill(t0, prompt) == first
        pin = [float(np.abs(t0.last_logits.double().cpu().numpy() - ref0.last_logits).max()
                     / np.abs(ref0.last_logits).max())]
        ts = []
        for ad in ads:
            t = tr.session(R.Adapter.from_oracle(ad, device="cuda"))
            t.copy_prefix(t0, len(prompt))
            ts.append(t)
        feed = [first, first]
        for step, want_toks in enumerate(oracle_toks):
            got = tr.decode_fused(ts, feed)
            for t, r in zip(ts, oracle_logits[step]):
                pin.append(float(np.abs(t.last_logits.double().cpu().numpy() - r).max() / np.abs(r).max()))
            assert got == want_toks
            feed = want_toks
        assert max(pin) <= 1e-4, pin
        del tr, t0, ts
        torch.cuda.empty_cache()
    k, v = sess[0].cache.rows(0, 0, sess[0].cache.position_count)
    rk = refs[0].k[0].reshape(k.shape)
    assert np.abs(k - rk).max() <= 2e-2 * np.abs(rk).max() + 1e-2
    print(f"8B-width worst relative logit error {worst:.3e}")
    for s in sess:
        s.close()
