"""The reference's module-level model API on the B200 kernels (paper_2603_13281_b200.model:
base_linear, adapted_linear, icarus_linear, layer_attention, block_forward,
decoder_block_readonly -- src/model.py:334-538), restating the reference's own model tests
(pkg/tests/test_model.py) on the GPU, plus: a model assembled from block_forward calls writes
exactly the KV bytes the engine's fused forward writes, and session.last_logits (computed on
demand from the kept final hidden) is bitwise the eagerly captured logits.

Structural identities are bitwise; values are bf16 operands with fp32 accumulation, checked
against the f64/f32 formula within a stated band.
"""

import numpy as np
import pytest

from oracle import icarus_oracle as O

pytestmark = pytest.mark.gpu
C1 = dict(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128, ffn_dim=1024,
          vocab_size=1024)
TOY = dict(num_layers=2, hidden_dim=8, num_heads=2, num_kv_heads=1, head_dim=4, ffn_dim=16,
           vocab_size=32)


def _mods():
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200 import kvpool as P
    from paper_2603_13281_b200 import model as M
    return E, P, M


def bf(a):
    return O.round_bf16(np.asarray(a, np.float32))


@pytest.fixture(scope="module")
def c1(cuda):
    E, P, M = _mods()
    shape = O.Shape(**C1)
    w = O.bf16_weights(O.init_base(shape, 0))
    cfg = M.ModelConfig(**C1)
    base = M.BaseWeights(cfg, w["embed"], [dict(l) for l in w["layers"]], w["final_gain"], w["lm_head"])
    agents = [M.AdapterSet(cfg, a["rank"], a["alpha"], M.DECODER_TARGETS,
                           [{t: M.LowRankPair(M.Param(p["a"]), M.Param(p["b"])) for t, p in per.items()}
                            for per in a["layers"]])
              for a in (O.bf16_adapter(x) for x in O.make_agents(shape, 2, seed=1))]
    rt = base.runtime(max_seqs=16, max_context=128, max_rows=64, adapter_slots=4, lora_rank=8)
    return base, agents, rt


# ------------------------------------------------------------------------ projections
def test_adapted_linear_zero_b_equals_base_bitwise(cuda):
    """pkg/tests/test_model.py:106-114."""
    E, P, M = _mods()
    cfg = M.ModelConfig(**TOY)
    rng = np.random.default_rng(5)
    x = M.Param(bf(rng.standard_normal((3, cfg.hidden_dim))))
    w = M.Param(bf(rng.standard_normal((cfg.hidden_dim, cfg.q_dim))))
    adapters = M.AdapterSet.init(cfg, seed=2)
    plain = M.base_linear(x, w).data
    adapted = M.adapted_linear(x, w, adapters.pair(0, "q"), adapters.scaling).data
    assert np.array_equal(plain, adapted)
    # and the projection itself is x @ W (bf16 operands are exact here, fp32 sums)
    assert np.allclose(plain, x.data.astype(np.float64) @ w.data.astype(np.float64), rtol=1e-5, atol=1e-5)


def test_icarus_linear_adapts_only_the_decoder_row(cuda):
    """pkg/tests/test_model.py:117-132: row 0 is the base projection bit for bit; row 1 adds
    scaling * (x1 A^T) B^T (U rounded to bf16 as in the decode step: band 1e-2)."""
    E, P, M = _mods()
    cfg = M.ModelConfig(**TOY)
    rng = np.random.default_rng(6)
    pair_in = bf(rng.standard_normal((2, cfg.hidden_dim)))
    w = M.Param(bf(rng.standard_normal((cfg.hidden_dim, cfg.q_dim))))
    adapters = M.AdapterSet.init(cfg, rank=2, seed=4)
    lr = adapters.pair(0, "q")
    lr.a.data = bf(lr.a.data)
    lr.b.data = bf(rng.standard_normal(lr.b.shape) / adapters.scaling) * np.float32(1.0)
    out = M.icarus_linear(M.Param(pair_in), w, lr, adapters.scaling).data
    plain = M.base_linear(M.Param(pair_in), w).data
    assert np.array_equal(out[0], plain[0])
    x1 = pair_in[1].astype(np.float64)
    want1 = x1 @ w.data + adapters.scaling * (x1 @ lr.a.data.T.astype(np.float64) @ lr.b.data.T)
    assert np.abs(out[1] - want1).max() <= 1e-2 * np.abs(want1).max() + 1e-3
    assert not np.array_equal(out[1], plain[1])


def test_icarus_linear_requires_a_pair(cuda):
    """pkg/tests/test_model.py:135-139."""
    E, P, M = _mods()
    from paper_2603_13281_b200.errors import ShapeError
    cfg = M.ModelConfig(**TOY)
    w = M.Param(np.ones((cfg.hidden_dim, cfg.q_dim), np.float32))
    with pytest.raises(ShapeError):
        M.icarus_linear(M.Param(np.ones((3, cfg.hidden_dim), np.float32)), w, None, 0.0)


def test_linear_rows_are_batch_invariant_at_llama_width(cuda):
    """A row's projection does not depend on the rows it shares the GEMM with (the reference's
    _mm property, tests/test_tensor.py:36-44), at d 4096 -> 14336 with a rank-16 term."""
    E, P, M = _mods()
    rng = np.random.default_rng(9)
    w = M.Param(bf(rng.standard_normal((4096, 1024)) / 64))
    pair = M.LowRankPair(M.Param(bf(rng.standard_normal((16, 4096)) / 64)),
                         M.Param(bf(rng.standard_normal((1024, 16)) * 0.05)))
    x = bf(rng.standard_normal((40, 4096)))
    many = M.adapted_linear(M.Param(x), w, pair, 2.0).data
    for i in (0, 17, 39):
        one = M.adapted_linear(M.Param(x[i:i + 1]), w, pair, 2.0).data
        assert np.array_equal(one[0], many[i])


# ------------------------------------------------------------------------ attention
def test_single_key_attention_returns_value_groups(c1):
    """pkg/tests/test_model.py:213-222 (one key: weight exactly 1)."""
    E, P, M = _mods()
    cfg = M.ModelConfig(**C1)
    rng = np.random.default_rng(4)
    q = bf(rng.standard_normal((1, cfg.q_dim)))
    k = bf(rng.standard_normal((1, cfg.kv_dim)))
    v = bf(rng.standard_normal((1, cfg.kv_dim)))
    out = M.layer_attention(M.Param(q), M.Param(k), M.Param(v), [0], cfg).data
    want = np.concatenate([v[0, :cfg.head_dim]] * cfg.num_heads)[None, :]
    assert np.array_equal(out, want)


def test_fused_double_head_call_equals_two_single_calls(c1):
    """pkg/tests/test_model.py:225-239: the 2H call == two H calls, bitwise."""
    E, P, M = _mods()
    cfg = M.ModelConfig(**C1)
    rng = np.random.default_rng(7)
    t = 37
    q_enc, q_dec = bf(rng.standard_normal((1, cfg.q_dim))), bf(rng.standard_normal((1, cfg.q_dim)))
    k, v = M.Param(bf(rng.standard_normal((t, cfg.kv_dim)))), M.Param(bf(rng.standard_normal((t, cfg.kv_dim))))
    fused = M.layer_attention(M.Param(np.concatenate([q_enc, q_dec], 1)), k, v, [t - 1], cfg).data
    enc = M.layer_attention(M.Param(q_enc), k, v, [t - 1], cfg).data
    dec = M.layer_attention(M.Param(q_dec), k, v, [t - 1], cfg).data
    assert np.array_equal(fused[:, :cfg.q_dim], enc)
    assert np.array_equal(fused[:, cfg.q_dim:], dec)
    # and the values are the reference attention's (bf16 output band)
    want = O.attention(np.concatenate([q_enc, q_dec], 1), k.data, v.data, [t - 1], O.Shape(**C1))
    assert np.abs(fused - want).max() <= 1e-2 * np.abs(want).max()


def test_attention_head_count_and_state_guards(c1):
    """pkg/tests/test_model.py:242-252."""
    E, P, M = _mods()
    from paper_2603_13281_b200.errors import ModeError, StateError
    cfg = M.ModelConfig(**C1)
    k = M.Param(np.ones((3, cfg.kv_dim), np.float32))
    v = M.Param(np.ones((3, cfg.kv_dim), np.float32))
    with pytest.raises(ModeError):
        M.layer_attention(M.Param(np.ones((1, 3 * cfg.q_dim), np.float32)), k, v, [0], cfg)
    with pytest.raises(StateError):
        M.layer_attention(M.Param(np.ones((1, cfg.q_dim), np.float32)), k, v, [3], cfg)
    empty = M.Param(np.ones((0, cfg.kv_dim), np.float32))
    with pytest.raises(StateError):
        M.layer_attention(M.Param(np.ones((1, cfg.q_dim), np.float32)), empty, empty, [0], cfg)


def test_causal_masking_hides_future_keys(c1):
    """pkg/tests/test_model.py:255-268: row p does not change when keys beyond p are
    dropped -- bitwise."""
    E, P, M = _mods()
    cfg = M.ModelConfig(**C1)
    rng = np.random.default_rng(8)
    t = 40
    q = bf(rng.standard_normal((t, cfg.q_dim)))
    k, v = bf(rng.standard_normal((t, cfg.kv_dim))), bf(rng.standard_normal((t, cfg.kv_dim)))
    full = M.layer_attention(M.Param(q), M.Param(k), M.Param(v), np.arange(t), cfg).data
    for p in (0, 2, 17, 33):
        row = M.layer_attention(M.Param(q[p:p + 1]), M.Param(k[:p + 1]), M.Param(v[:p + 1]), [p], cfg).data
        assert np.array_equal(full[p:p + 1], row), p
    want = O.attention(q, k, v, np.arange(t), O.Shape(**C1))
    assert np.abs(full - want).max() <= 1e-2 * np.abs(want).max()


# ------------------------------------------------------------------------ blocks
def _cache(M, base, rt, cap=64):
    return M.KvCacheTensor(base.config, cap, arena=rt.arena)


def _prefill_layers(M, base, tokens, cache, ledger=None, upto=None):
    x = M.Param(base.embed.data[np.asarray(tokens)].copy())
    for layer in range(base.config.num_layers if upto is None else upto):
        x = M.block_forward(x, layer, base, None, cache, "prefill", np.arange(len(tokens)), ledger)
    return x


def test_block_prefill_then_decode_ledger_counts(c1):
    """pkg/tests/test_model.py:280-297: 7 / 7 / 5 parameter reads."""
    E, P, M = _mods()
    from paper_2603_13281_b200.metrics import Ledger
    base, agents, rt = c1
    cache = _cache(M, base, rt)
    ledger = Ledger()
    _prefill_layers(M, base, [1, 2, 3], cache, ledger, upto=1)
    assert ledger.param_matrix_reads == 7
    pair = M.Param(np.vstack([base.embed.data[4], base.embed.data[5]]))
    ledger2 = Ledger()
    M.block_forward(pair, 0, base, agents[0], cache, "decode", [3], ledger2)
    assert ledger2.param_matrix_reads == 7
    ledger3 = Ledger()
    M.decoder_block_readonly(M.Param(base.embed.data[5:6].copy()), 0, base, agents[0], cache, 3, ledger3)
    assert ledger3.param_matrix_reads == 5
    assert cache.length(0) == 4 and cache.length(1) == 0
    cache.release()


def test_block_decode_cache_ignores_decoder_row(c1):
    """pkg/tests/test_model.py:300-317: the decoder row cannot change the cache bytes."""
    E, P, M = _mods()
    base, agents, rt = c1
    outs, prints = [], []
    for row1_token in (9, 21):
        cache = _cache(M, base, rt)
        _prefill_layers(M, base, [1, 2, 3], cache, upto=1)
        x = M.Param(np.vstack([base.embed.data[4], base.embed.data[row1_token]]))
        outs.append(M.block_forward(x, 0, base, agents[0], cache, "decode", [3]).data)
        prints.append(cache.fingerprint())
        cache.release()
    assert prints[0] == prints[1]
    assert np.array_equal(outs[0][0], outs[1][0])
    assert not np.array_equal(outs[0][1], outs[1][1])


def test_block_mode_and_position_guards(c1):
    """pkg/tests/test_model.py:320-336."""
    E, P, M = _mods()
    from paper_2603_13281_b200.errors import ModeError, ShapeError, StateError
    base, agents, rt = c1
    cfg = base.config
    cache = _cache(M, base, rt)
    _prefill_layers(M, base, [1, 2], cache, upto=1)
    pair = M.Param(np.ones((2, cfg.hidden_dim), np.float32))
    with pytest.raises(ModeError):
        M.block_forward(pair, 0, base, None, cache, "train", [2])
    with pytest.raises(StateError):
        M.block_forward(pair, 0, base, None, cache, "decode", [5])
    with pytest.raises(ShapeError):
        M.block_forward(M.Param(np.ones((3, cfg.hidden_dim), np.float32)), 0, base, None, cache, "decode", [2])
    with pytest.raises(StateError):
        M.decoder_block_readonly(M.Param(np.ones((1, cfg.hidden_dim), np.float32)), 0, base, None, cache, 5)
    cache.release()


def test_blocks_compose_to_the_engine_forward_bitwise(c1):
    """L block_forward calls == the engine's fused forward: same K/V bytes for prefill and for
    an adapted fused decode step (the per-layer entry runs the same kernels), and the decoder
    row's final hidden gives the engine's logits."""
    E, P, M = _mods()
    base, agents, rt = c1
    cfg = base.config
    prompt = [int(t) for t in np.random.default_rng(3).integers(1, 1024, 21)]
    s = E.new_session(base, agents[1], 64, runtime=rt)
    E.prefill(s, prompt)
    cache = _cache(M, base, rt)
    _prefill_layers(M, base, prompt, cache)
    assert cache.fingerprint() == s.cache.fingerprint()
    tok = 77
    E.decode_step_fused(s, tok)
    x = M.Param(np.vstack([base.embed.data[tok]] * 2))
    for layer in range(cfg.num_layers):
        x = M.block_forward(x, layer, base, agents[1], cache, "decode", [len(prompt)])
    assert cache.fingerprint() == s.cache.fingerprint()
    h = x.data[1].astype(np.float64)
    h = h / np.sqrt(np.mean(h * h) + cfg.rms_eps)
    want = h @ base.lm_head.data.astype(np.float64)
    assert np.abs(s.last_logits - want).max() <= 1e-2 * np.abs(want).max()
    s.close()
    cache.release()


# ------------------------------------------------------------------------ last_logits
def test_lazy_last_logits_equal_captured_and_survive_commit_probes(c1):
    """session.last_logits is always available (engine.py:127, 191, 214), computed on demand
    from the kept final hidden -- bitwise the logits an eager (capture_logits) forward writes;
    base_next_token_at's probe rows do not disturb it; positions the session did not compute
    raise StateError (engine.py:280-282)."""
    E, P, M = _mods()
    from paper_2603_13281_b200.errors import StateError
    base, agents, rt = c1
    prompt = [int(t) for t in np.random.default_rng(5).integers(1, 1024, 37)]
    lazy = [E.new_session(base, a, 96, runtime=rt) for a in (agents[0], None)]
    eager = [E.new_session(base, a, 96, runtime=rt, capture_logits=True) for a in (agents[0], None)]
    pool = P.KvCachePool(base.config, budget_bytes=1 << 26, mode="icarus")
    t_l = [E.prefill(lazy[0], prompt, pool=pool), E.prefill(lazy[1], prompt)]
    t_e = [E.prefill(s, prompt) for s in eager]
    assert t_l == t_e
    for a, b in zip(lazy, eager):
        assert a.last_logits.tobytes() == b.last_logits.tobytes()
    for _ in range(3):
        t_l = E.decode_step_batch(lazy, t_l)
        t_e = E.decode_step_batch(eager, t_e)
        assert t_l == t_e
        E.base_next_token_at(lazy[0], 5)  # a probe row at a computed prefill position
        for a, b in zip(lazy, eager):
            assert a.last_logits.tobytes() == b.last_logits.tobytes()
    seq_tok = E.decode_step_sequential(lazy[0], t_l[0])
    assert int(np.argmax(lazy[0].last_logits)) == seq_tok
    # a session that reuses the pooled prefix did not compute those positions
    pool.commit(None, prompt, lazy[0].cache, next_token_fn=lambda p: E.base_next_token_at(lazy[0], p))
    hit = E.new_session(base, agents[1], 96, runtime=rt)
    E.prefill(hit, prompt, pool=pool)
    assert hit.ledger.prefix_hit_tokens == 32
    with pytest.raises(StateError):
        E.base_next_token_at(hit, 3)
    assert E.base_next_token_at(hit, 36) == E.base_next_token_at(lazy[0], 36)
    for s in lazy + eager + [hit]:
        s.close()
