"""Generate golden vectors by running the UNMODIFIED reference `icarus` package.

Only runnable where /root/reference exists (the build container); the outputs are
committed next to this script and are what tests/ compare against on any box.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Produces
  toy_decode.npz      reference toy config (tests/test_engine.py:15-32), f32 weights:
                      prefill + 10 fused decode steps, logits bytes -> pins the oracle BITWISE
  c1_decode.npz       C1 (BASELINE.json configs[0]) with bf16-representable weights and the
                      2 agents of make_agents(cfg, 2, seed=1): agent0 prefills a 128-token
                      prompt through an icarus-mode pool and decodes 32 tokens, commits;
                      agent1 hits the full prefix and decodes 32 tokens. Logits per step,
                      tokens, agent0's K/V cache, pool stats.
  pool_scenarios.json random op sequences on KvCachePool (both modes, both eviction
                      policies) with every return value, exception and stats() snapshot.
  chain_hash.json     chain_hash known answers.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from icarus import engine as E  # noqa: E402
from icarus.errors import IcarusError  # noqa: E402
from icarus.kvpool import BLOCK_TOKENS, KvCachePool, chain_hash  # noqa: E402
from icarus.model import (AdapterSet, BaseWeights, KvCacheTensor, ModelConfig,  # noqa: E402
                          init_base)
from icarus.simulate import make_agents  # noqa: E402


def round_bf16(x):
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


# ----------------------------------------------------------------------------- toy
def toy():
    cfg = ModelConfig(num_layers=2, hidden_dim=8, num_heads=2, num_kv_heads=1, head_dim=4,
                      ffn_dim=16, vocab_size=32)
    base = init_base(cfg, 0)
    ad = AdapterSet.init(cfg, seed=1)
    rng = np.random.default_rng(101)
    for per in ad.layers:
        for pair in per.values():
            pair.b.data = (rng.standard_normal(pair.b.shape) * 0.1).astype(cfg.dtype)
    prompt = [3, 1, 4, 1, 5]
    s = E.new_session(base, ad, 64)
    tok = E.prefill(s, prompt)
    toks = [tok]
    logits = [s.last_logits.copy()]
    for _ in range(10):
        tok = E.decode_step_fused(s, tok)
        toks.append(tok)
        logits.append(s.last_logits.copy())
    k = np.stack([s.cache._k[l][:s.cache.length(l)] for l in range(cfg.num_layers)])
    v = np.stack([s.cache._v[l][:s.cache.length(l)] for l in range(cfg.num_layers)])
    np.savez_compressed(HERE / "toy_decode.npz", prompt=np.asarray(prompt), tokens=np.asarray(toks),
                        logits=np.stack(logits), k=k, v=v,
                        fingerprint=np.frombuffer(s.cache.fingerprint().encode(), np.uint8))
    print("toy tokens", toks)


# ----------------------------------------------------------------------------- C1
C1 = dict(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128, ffn_dim=1024,
          vocab_size=1024)


def c1():
    cfg = ModelConfig(**C1)
    raw = init_base(cfg, 0)
    layers = []
    for lw in raw.layers:
        layers.append({name: (round_bf16(getattr(lw, name).data) if "gain" not in name
                              else getattr(lw, name).data.copy())
                       for name in lw._fields})
    base = BaseWeights(cfg, round_bf16(raw.embed.data), layers, raw.final_gain.data.copy(),
                       round_bf16(raw.lm_head.data))
    agents = make_agents(cfg, 2, seed=1)
    for ad in agents:
        for per in ad.layers:
            for pair in per.values():
                pair.a.data = round_bf16(pair.a.data)
                pair.b.data = round_bf16(pair.b.data)
    prompt = [int(t) for t in np.random.default_rng(0).integers(1, cfg.vocab_size, 128)]
    pool = KvCachePool(cfg, budget_bytes=64 << 20, mode="icarus")
    out = {"prompt": np.asarray(prompt)}
    for i, ad in enumerate(agents):
        s = E.new_session(base, ad, 512)
        tok = E.prefill(s, prompt, pool=pool, namespace=None, reader=f"agent{i}")
        toks = [tok]
        if s.last_logits is not None:
            out[f"a{i}_prefill_logits"] = s.last_logits.copy()
        logits = []
        for _ in range(32):
            tok = E.decode_step_fused(s, tok)
            toks.append(tok)
            logits.append(s.last_logits.copy())
        out[f"a{i}_tokens"] = np.asarray(toks)
        out[f"a{i}_logits"] = np.stack(logits)
        out[f"a{i}_hit"] = np.asarray(s.ledger.prefix_hit_tokens)
        out[f"a{i}_ledger"] = np.asarray([s.ledger.prefill_tokens, s.ledger.prefix_hit_tokens,
                                          s.ledger.decode_steps, s.ledger.param_passes,
                                          s.ledger.param_matrix_reads, s.ledger.kv_read_events,
                                          s.ledger.kv_bytes_read, s.ledger.kv_bytes_written])
        if i == 0:
            n = s.cache.position_count
            out["a0_k"] = np.stack([s.cache._k[l][:n] for l in range(cfg.num_layers)])
            out["a0_v"] = np.stack([s.cache._v[l][:n] for l in range(cfg.num_layers)])
            pool.commit(None, prompt + toks[:-1], s.cache,
                        next_token_fn=lambda p, s=s: E.base_next_token_at(s, p), creator="agent0")
        if s.borrowed_chain:
            pool.release(s.borrowed_chain)
    out["pool_stats"] = np.frombuffer(json.dumps(pool.stats(), sort_keys=True).encode(), np.uint8)
    np.savez_compressed(HERE / "c1_decode.npz", **out)
    print("c1 a0", out["a0_tokens"][:8], "a1", out["a1_tokens"][:8])


# ----------------------------------------------------------------------------- pool
POOL_CFG = dict(num_layers=2, hidden_dim=8, num_heads=2, num_kv_heads=1, head_dim=4, ffn_dim=16,
                vocab_size=32)


def filled_cache(cfg, n, seed):
    cache = KvCacheTensor(cfg, max(n, 1))
    rng = np.random.default_rng(seed)
    shape = (n, cfg.num_kv_heads, cfg.head_dim)
    if n:
        for layer in range(cfg.num_layers):
            cache.append_block(layer, rng.standard_normal(shape).astype(cfg.dtype),
                               rng.standard_normal(shape).astype(cfg.dtype), source_branch=0)
    return cache


def gen_ops(seed: int, n_ops: int, multi_ns: bool):
    """Random op program over a few shared prefixes (hits, dedups, divergence, eviction)."""
    rng = np.random.default_rng(seed)
    prefixes = [list(map(int, rng.integers(0, 32, 64))) for _ in range(3)]
    ops = []
    open_chains = 0
    for _ in range(n_ops):
        kind = rng.choice(["commit", "lookup", "release", "evict"], p=[0.4, 0.35, 0.15, 0.1])
        ns = f"agent{int(rng.integers(0, 3))}" if multi_ns else None
        who = f"agent{int(rng.integers(0, 3))}"
        if kind in ("commit", "lookup"):
            p = prefixes[int(rng.integers(0, 3))]
            cut = int(rng.integers(1, 64))
            toks = p[:cut] + list(map(int, rng.integers(0, 32, int(rng.integers(0, 24)))))
            if kind == "commit":
                ops.append({"op": "commit", "ns": ns, "tokens": toks, "creator": who,
                            "seed": int(rng.integers(0, 1 << 30)), "next": bool(rng.random() < 0.5)})
            else:
                ops.append({"op": "lookup", "ns": ns, "tokens": toks, "reader": who})
                open_chains += 1
        elif kind == "release" and open_chains:
            ops.append({"op": "release", "which": int(rng.integers(0, open_chains))})
        elif kind == "evict":
            ops.append({"op": "evict", "blocks": int(rng.integers(1, 4))})
    return ops


def run_ops(cfg, pool, ops):
    chains = []
    results = []
    bb = pool.block_nbytes
    for op in ops:
        rec = {}
        try:
            if op["op"] == "commit":
                cache = filled_cache(cfg, len(op["tokens"]), op["seed"])
                fn = (lambda p: (p * 7 + 3) % 32) if op["next"] else None
                blocks = pool.commit(op["ns"], op["tokens"], cache, next_token_fn=fn,
                                     creator=op["creator"])
                rec["blocks"] = [b.block_id for b in blocks]
                rec["hashes"] = [str(b.hash) for b in blocks]
                rec["next"] = [b.next_token for b in blocks]
            elif op["op"] == "lookup":
                matched, chain = pool.lookup(op["ns"], op["tokens"], reader=op["reader"])
                chains.append(chain)
                rec["matched"] = matched
                rec["blocks"] = [b.block_id for b in chain]
            elif op["op"] == "release":
                live = [c for c in chains if c is not None]
                if live:
                    idx = op["which"] % len(live)
                    target = live[idx]
                    pool.release(target)
                    chains[chains.index(target)] = None
                rec["released"] = True
            elif op["op"] == "evict":
                rec["freed"] = pool.evict(op["blocks"] * bb)
        except IcarusError as exc:
            rec["error"] = type(exc).__name__
        rec["stats"] = pool.stats()
        rec["residency"] = sorted([b.block_id, b.residency, b.ref_count]
                                  for b in pool._index.values())
        results.append(rec)
    return results


def pool_scenarios():
    cfg = ModelConfig(**POOL_CFG)
    scen = []
    variants = [("baseline", "recompute", 0, True, 12), ("icarus", "recompute", 0, False, 12),
                ("baseline", "swap", 6, True, 10), ("icarus", "swap", 4, False, 8),
                ("icarus", "recompute", 0, False, 6)]
    for i, (mode, ev, swap_blocks, multi, budget_blocks) in enumerate(variants):
        ops = gen_ops(1000 + i, 120, multi)
        bb = 16 * cfg.kv_bytes_per_token
        pool = KvCachePool(cfg, budget_blocks * bb, mode, eviction=ev,
                           swap_budget_bytes=swap_blocks * bb)
        res = run_ops(cfg, pool, ops)
        scen.append({"mode": mode, "eviction": ev, "budget_blocks": budget_blocks,
                     "swap_blocks": swap_blocks, "ops": ops, "results": res})
    (HERE / "pool_scenarios.json").write_text(json.dumps({"config": POOL_CFG, "scenarios": scen}))
    print("pool scenarios", len(scen))


def hashes():
    rng = np.random.default_rng(5)
    cases = []
    parent = 0
    for _ in range(8):
        chunk = [int(t) for t in rng.integers(0, 128256, BLOCK_TOKENS)]
        h = chain_hash(parent, tuple(chunk))
        cases.append({"parent": str(parent), "chunk": chunk, "hash": str(h)})
        parent = h
    (HERE / "chain_hash.json").write_text(json.dumps(cases))


if __name__ == "__main__":
    toy()
    hashes()
    pool_scenarios()
    c1()
