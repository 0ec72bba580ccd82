"""Batched multi-agent serving driver over the fused multi-model decode step (SURVEY.md §8(f)-2,
BASELINE.json configs[2] "C3" and configs[4] "C5").

The reference serves one request turn at a time through a FIFO simulator priced by a cost
model (`simulate.run`, src/simulate.py:254-364; continuous batching and multi-GPU placement
are its non-goals). This driver keeps its workload semantics -- the
`generate_workload` structure stream (src/simulate.py:114-160: turns, question / observation /
output lengths drawn uniformly from one `SeedSequence([seed, 0])` stream), cross-model prefix
reuse through the pool between turns (src/simulate.py:306-335: lookup, decode, commit with the
base chunk-end token, release), `RunReport`-style counters and nearest-rank P95
(src/simulate.py:226-231) -- and replaces simulated time with real continuous batching: every
live turn of every request advances in ONE fused forward per step (encoder + decoder row per
session, each session its own adapter, KV shared through the pool); new turns join as soon as
their context is ready, their prefill riding in the same forward (`engine.step_batch`);
finished turns commit their blocks and release their pins.

C3 extension (SURVEY.md §8 "C3"): all requests share one `prefix_len`-token prefix that is
prefilled once by the base model and committed before serving, so every first turn is a
cross-model prefix hit; turn j of request r is routed to adapter (r + j) mod n so all n
adapters are live (the reference's round-robin, src/simulate.py:103-111, keys on j only).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import engine as E
from .dist import p95_nearest_rank
from .errors import ConfigError


@dataclass(frozen=True)
class WorkflowConfig:
    requests: int = 64
    num_agents: int = 8
    prefix_len: int = 8192
    question_min: int = 64
    question_max: int = 128
    turns_min: int = 2
    turns_max: int = 4
    output_min: int = 64
    output_max: int = 128
    obs_min: int = 32
    obs_max: int = 64
    seed: int = 0
    vocab_low: int = 1
    max_batch: int = 64          # sessions advanced per fused step

    def validate(self) -> None:
        for lo, hi, name in ((self.question_min, self.question_max, "question"),
                             (self.turns_min, self.turns_max, "turns"),
                             (self.output_min, self.output_max, "output"),
                             (self.obs_min, self.obs_max, "observation")):
            if lo < 1 or hi < lo:
                raise ConfigError(f"{name} length range [{lo}, {hi}] is invalid")
        if self.requests < 1 or self.num_agents < 1 or self.max_batch < 1 or self.prefix_len < 0:
            raise ConfigError("requests, num_agents and max_batch must be positive")


@dataclass(frozen=True)
class Turn:
    agent: int
    new_tokens: tuple[int, ...]   # question (turn 0) or observation (later turns)
    output_len: int


@dataclass(frozen=True)
class Request:
    rid: int
    turns: tuple[Turn, ...]


def make_workload(cfg: WorkflowConfig, vocab_size: int) -> tuple[tuple[int, ...], list[Request]]:
    """(shared prefix, requests), deterministic in cfg.seed (src/simulate.py:114-160 streams)."""
    cfg.validate()
    if vocab_size <= cfg.vocab_low + 1:
        raise ConfigError(f"vocab {vocab_size} too small for token draws")
    structure = np.random.default_rng(np.random.SeedSequence([cfg.seed, 0]))
    prefix_rng = np.random.default_rng(np.random.SeedSequence([cfg.seed, 2]))

    def draw(n: int) -> tuple[int, ...]:
        return tuple(int(t) for t in structure.integers(cfg.vocab_low, vocab_size, n))

    prefix = tuple(int(t) for t in prefix_rng.integers(cfg.vocab_low, vocab_size, cfg.prefix_len))
    reqs = []
    for rid in range(cfg.requests):
        n_turns = int(structure.integers(cfg.turns_min, cfg.turns_max + 1))
        turns = []
        for j in range(n_turns):
            agent = (rid + j) % cfg.num_agents
            if j == 0:
                new = draw(int(structure.integers(cfg.question_min, cfg.question_max + 1)))
            else:
                new = draw(int(structure.integers(cfg.obs_min, cfg.obs_max + 1)))
            out = int(structure.integers(cfg.output_min, cfg.output_max + 1))
            turns.append(Turn(agent, new, out))
        reqs.append(Request(rid, tuple(turns)))
    return prefix, reqs


def max_context_tokens(prefix: Sequence[int], reqs: Sequence[Request]) -> int:
    worst = 0
    for r in reqs:
        n = len(prefix)
        for t in r.turns:
            n += len(t.new_tokens) + t.output_len
        worst = max(worst, n)
    return worst


@dataclass
class ServeReport:
    """RunReport-shaped summary (src/simulate.py:183-231), measured on the device."""
    completed: int = 0
    turns: int = 0
    latencies_ms: list = field(default_factory=list)
    p95_latency_ms: float = 0.0
    wall_s: float = 0.0
    decode_steps: int = 0          # fused steps (each advances every live session)
    decoder_tokens: int = 0        # tokens emitted by decode steps (prefill tokens excluded)
    decode_tok_s: float = 0.0
    prefill_tokens: int = 0
    prefix_hit_tokens: int = 0
    cross_model_hit_tokens: int = 0
    max_live: int = 0
    outputs: dict = field(default_factory=dict)   # (rid, turn) -> emitted tokens


@dataclass
class _Live:
    req: Request
    turn: int
    context: list
    session: E.GenerationSession
    out: list


def serve(base, adapters: Sequence, pool, prefix: Sequence[int], reqs: Sequence[Request],
          cfg: WorkflowConfig, max_context: int, runtime=None, ledger=None) -> ServeReport:
    """Continuous-batching multi-agent serving; returns a ServeReport. All requests are present
    at t = 0 (closed batch); the shared prefix must already be committed in `pool`. `ledger`
    (optional) is shared by every session, as the reference's run() shares one
    (src/simulate.py:277, 318-319). In a "baseline"-mode pool every agent reads and commits
    in its own namespace (src/simulate.py:313)."""
    rep = ServeReport()
    stats0 = pool.stats()
    live: list[_Live] = []
    pending = list(reqs)       # requests whose next turn has not started
    contexts = {r.rid: list(prefix) for r in reqs}
    next_turn = {r.rid: 0 for r in reqs}
    t0 = time.perf_counter()

    def space(agent: int):
        return f"agent{agent}" if pool.mode == "baseline" else None

    def open_turns(reqs_: list) -> list:
        """Open the next turn of each request (sessions not yet prefilled)."""
        out = []
        for req in reqs_:
            turn = req.turns[next_turn[req.rid]]
            ctx = contexts[req.rid] + list(turn.new_tokens)
            s = E.new_session(base, adapters[turn.agent], max_context, runtime=runtime,
                              ledger=ledger)
            out.append(_Live(req, next_turn[req.rid], ctx, s, []))
        return out

    def finish_turn(lv: _Live) -> None:
        s, turn = lv.session, lv.req.turns[lv.turn]
        covered = lv.context + lv.out[:-1]   # the last emitted token has no KV yet
        pool.commit(space(turn.agent), covered, s.cache,
                    next_token_fn=lambda p: E.base_next_token_at(s, p), creator=f"agent{turn.agent}")
        if s.borrowed_chain:
            pool.release(s.borrowed_chain)
            s.borrowed_chain = []
        s.close()
        rep.outputs[(lv.req.rid, lv.turn)] = list(lv.out)
        contexts[lv.req.rid] = lv.context + lv.out
        next_turn[lv.req.rid] = lv.turn + 1
        rep.turns += 1
        if next_turn[lv.req.rid] == len(lv.req.turns):
            rep.completed += 1
            rep.latencies_ms.append((time.perf_counter() - t0) * 1e3)
        else:
            pending.append(lv.req)

    while live or pending:
        starting = []
        while pending and len(live) + len(starting) < cfg.max_batch:
            starting.append(pending.pop(0))
        new = open_turns(starting)
        # a turn whose output is a single token is complete after prefill
        done = [lv for lv in live if len(lv.out) >= lv.req.turns[lv.turn].output_len]
        active = [lv for lv in live if len(lv.out) < lv.req.turns[lv.turn].output_len]
        if active or new:
            # one decode step of the running turns, the new turns' prefill riding in the same
            # forward (engine.step_batch): the base weights stream once for both
            nxt, firsts = E.step_batch([lv.session for lv in active], [lv.out[-1] for lv in active],
                                       [lv.session for lv in new], [lv.context for lv in new],
                                       pool=pool,
                                       namespace=[space(lv.req.turns[lv.turn].agent) for lv in new],
                                       readers=[f"agent{lv.req.turns[lv.turn].agent}" for lv in new])
            if active:
                rep.decode_steps += 1
                rep.decoder_tokens += len(active)
            for lv, t in zip(active, nxt):
                lv.out.append(t)
                if len(lv.out) >= lv.req.turns[lv.turn].output_len:
                    done.append(lv)
            for lv, first in zip(new, firsts):
                lv.out.append(first)
                rep.prefill_tokens += lv.session.ledger.prefill_tokens
                rep.prefix_hit_tokens += lv.session.ledger.prefix_hit_tokens
                live.append(lv)
        rep.max_live = max(rep.max_live, len(live))
        for lv in done:
            live.remove(lv)
            finish_turn(lv)
    rep.wall_s = time.perf_counter() - t0
    rep.decode_tok_s = rep.decoder_tokens / rep.wall_s if rep.wall_s > 0 else 0.0
    rep.p95_latency_ms = p95_nearest_rank(rep.latencies_ms)
    stats1 = pool.stats()
    rep.cross_model_hit_tokens = int(stats1.get("cross_model_hit_tokens", 0)) - int(
        stats0.get("cross_model_hit_tokens", 0))
    return rep


def warm_prefix(base, pool, prefix: Sequence[int], max_context: int, runtime=None) -> int:
    """Prefill the shared prefix once with the bare base model and commit its full blocks
    (every later turn's lookup hits them); returns the committed token count."""
    if not prefix:
        return 0
    s = E.new_session(base, None, max_context, runtime=runtime)
    E.prefill(s, list(prefix), pool=pool, namespace=None, reader="prefix")
    pool.commit(None, list(prefix), s.cache, next_token_fn=lambda p: E.base_next_token_at(s, p),
                creator="prefix")
    if s.borrowed_chain:
        pool.release(s.borrowed_chain)
    s.close()
    return (len(prefix) // 16) * 16
