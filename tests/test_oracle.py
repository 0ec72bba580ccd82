"""Pin the CPU oracle against golden vectors produced by the unmodified reference.

These run on CPU (no GPU marker). If the oracle drifted from the reference by a single
bit, the GPU parity tests that use it as the checker would be meaningless.
"""

import json
from pathlib import Path

import numpy as np

from oracle import icarus_oracle as O

GOLD = Path(__file__).resolve().parent / "golden"

TOY = O.Shape(num_layers=2, hidden_dim=8, num_heads=2, num_kv_heads=1, head_dim=4, ffn_dim=16,
              vocab_size=32)
C1 = O.Shape(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128,
             ffn_dim=1024, vocab_size=1024)


def live_adapter(cfg, seed=1, scale=0.1):
    """tests/test_engine.py:26-32 (reference live_adapters)."""
    ad = O.init_adapter(cfg, seed)
    rng = np.random.default_rng(seed + 100)
    for per in ad["layers"]:
        for pair in per.values():
            pair["b"] = (rng.standard_normal(pair["b"].shape) * scale).astype(np.float32)
    return ad


def test_toy_fused_decode_is_bitwise_reference():
    g = np.load(GOLD / "toy_decode.npz")
    s = O.Session(TOY, O.init_base(TOY, 0), live_adapter(TOY))
    toks = [s.prefill(list(g["prompt"]))]
    logits = [s.last_logits]
    for _ in range(10):
        toks.append(s.decode_fused(toks[-1]))
        logits.append(s.last_logits)
    assert toks == list(g["tokens"])
    assert np.stack(logits).tobytes() == g["logits"].tobytes()
    assert np.stack(s.k).tobytes() == g["k"].reshape(2, -1, 4).tobytes()
    assert np.stack(s.v).tobytes() == g["v"].reshape(2, -1, 4).tobytes()


def test_c1_two_agents_bitwise_reference():
    g = np.load(GOLD / "c1_decode.npz")
    w = O.bf16_weights(O.init_base(C1, 0))
    agents = [O.bf16_adapter(a) for a in O.make_agents(C1, 2, seed=1)]
    prompt = list(g["prompt"])
    s0 = O.Session(C1, w, agents[0])
    first = s0.prefill(prompt)
    assert s0.last_logits.tobytes() == g["a0_prefill_logits"].tobytes()
    toks, logits = [first], []
    for _ in range(32):
        toks.append(s0.decode_fused(toks[-1]))
        logits.append(s0.last_logits)
    assert toks == list(g["a0_tokens"])
    assert np.stack(logits).tobytes() == g["a0_logits"].tobytes()
    n = s0.length
    assert np.stack(s0.k).tobytes() == g["a0_k"].reshape(2, n, -1).tobytes()
    # agent1: full 128-token prefix hit -> installs agent0's prompt K/V and emits the
    # stored chunk-end base token (src/engine.py:135-139)
    s1 = O.Session(C1, w, agents[1])
    s1.install_prefix([k[:128] for k in s0.k], [v[:128] for v in s0.v])
    toks1 = [s0.base_next_token_at(127)]
    logits1 = []
    for _ in range(32):
        toks1.append(s1.decode_fused(toks1[-1]))
        logits1.append(s1.last_logits)
    assert toks1 == list(g["a1_tokens"])
    assert np.stack(logits1).tobytes() == g["a1_logits"].tobytes()


def test_chain_hash_known_answers():
    for case in json.loads((GOLD / "chain_hash.json").read_text()):
        assert O.chain_hash(int(case["parent"]), case["chunk"]) == int(case["hash"])


def test_bf16_rounding_is_round_to_nearest_even():
    import torch
    x = np.random.default_rng(0).standard_normal(4096).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    assert O.round_bf16(x).tobytes() == ref.tobytes()
