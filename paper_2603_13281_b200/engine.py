"""Generation sessions on the B200: prefill, the fused multi-model decode step, generate.

Drop-in for the reference's src/engine.py (same names, arguments, guards, ledger
arithmetic and error classes). Semantics carried over exactly:
  * prefill is encoder-only work and emits the BASE model's greedy token (engine.py:84-153),
    reusing the longest pooled block prefix and computing only the suffix;
  * a fused step runs the encoder row (base weights, writes K/V for `pos` before
    attention) and the decoder row (base + LoRA, predicts the next token) in ONE pass
    (engine.py:179-193, model.py:480-506);
  * greedy argmax, lowest id on ties (engine.py:75-76).

B200 generalisation: `decode_step_batch(sessions, tokens)` advances many sessions --
each with its own adapter -- in one forward over 2N token rows, with sessions that share
a prompt reading the same KV pages. The single-session calls are batch-of-one wrappers.
All compute goes through runtime.Runtime.forward (the C ABI); there is no CPU path.
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

from .errors import (CapacityError, ConfigError, ContractViolationError, ModeError,
                     StateError)
from .metrics import Ledger
from .model import BLOCK_TOKENS, DECODER_TARGETS, AdapterSet, BaseWeights, KvCacheTensor


class GenerationSession:
    """One sequence in flight: block-table row, page-backed cache, counters, predictions.

    `base_next` maps a computed position to the base model's greedy next token (the
    encoder row's argmax) -- what the reference derives from `final_hidden` for chunk-end
    commits (engine.py:274-284).

    `last_logits` keeps the reference contract (engine.py:127, 191, 214, 232: the logits of
    the last emitted token, None after a stored full-prefix hit) without paying for them on
    every step: each emitting forward keeps the row's final hidden state on the device (one
    slot per sequence and row kind), and the first read of `last_logits` runs the LM head
    over it -- the same GEMM over the same inputs as the fused step, so the values are
    bitwise those the step would have produced. `capture_logits=True` computes them eagerly
    inside every forward instead. A closed session keeps only logits already read."""

    def __init__(self, base: BaseWeights, adapter: Optional[AdapterSet], max_context: int,
                 ledger: Optional[Ledger] = None, runtime=None, capture_logits: bool = False):
        if adapter is not None:
            bad = set(adapter.targets) - set(DECODER_TARGETS)
            if bad:
                raise ContractViolationError(
                    f"adapter targets {sorted(bad)} cannot ride a shared cache; "
                    f"decoder-side targets are {DECODER_TARGETS}")
            if adapter.config != base.config:
                raise ConfigError("adapter was built for a different model config")
        if max_context < 1:
            raise ConfigError(f"max_context must be positive, got {max_context}")
        self.runtime = runtime if runtime is not None else base.runtime()
        if max_context > self.runtime.max_context:
            raise ConfigError(f"max_context {max_context} exceeds the runtime's "
                              f"{self.runtime.max_context}")
        self.base = base
        self.adapter = adapter
        self.config = base.config
        self.max_context = max_context
        self.ledger = ledger if ledger is not None else Ledger()
        self.capture_logits = capture_logits
        self.adapter_slot = self.runtime.slots.slot_of(adapter) if adapter is not None else -1
        self.seq = self.runtime.acquire_seq()
        self._bt_len = -1  # pages mirrored into the block table row (-1: row not written yet)
        self.cache = KvCacheTensor(base.config, max_context, arena=self.runtime.arena)
        self.prompt: list[int] = []
        self.produced: list[int] = []
        self.base_next: dict[int, int] = {}
        self._ll: Optional[np.ndarray] = None
        self._ll_kind: Optional[int] = None  # row kind whose stored hidden is pending
        self._computed: list = []  # [lo, hi) position ranges this session computed itself
        self.borrowed_chain: list = []
        self._prefilled = False
        self._closed = False

    @property
    def last_logits(self) -> Optional[np.ndarray]:
        if self._ll_kind is not None and not self._closed:
            lg = self.runtime.seq_logits([2 * self.seq + self._ll_kind])
            self._ll = lg[0].cpu().numpy()
            self._ll_kind = None
        return self._ll

    @last_logits.setter
    def last_logits(self, value) -> None:
        self._ll = value
        self._ll_kind = None

    def _logits_pending(self, kind: int) -> None:
        """The last forward kept this session's row of `kind` in the hidden store."""
        self._ll = None
        self._ll_kind = kind

    def _set_logits(self, lg, row: int, kind: int) -> None:
        if self.capture_logits and lg is not None:
            self.last_logits = _logits_np(lg, row)
        else:
            self._logits_pending(kind)

    def _note_computed(self, lo: int, hi: int) -> None:
        if self._computed and self._computed[-1][1] == lo:
            self._computed[-1][1] = hi
        else:
            self._computed.append([lo, hi])

    def computed(self, pos: int) -> bool:
        """Did this session compute position `pos` itself (the reference's final_hidden)?"""
        return any(lo <= pos < hi for lo, hi in self._computed)

    def close(self) -> None:
        """Return the sequence slot and this session's page references."""
        if self._closed:
            return
        self._ll_kind = None
        self._closed = True
        self.cache.release()
        self.runtime.release_seq(self.seq)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _sync_block_table(self) -> None:
        self.runtime.set_pages(self.seq, self.cache.pages)
        self._bt_len = len(self.cache.pages)

    def _sync_appended_pages(self) -> None:
        """Decode steps only ever append pages: mirror just the new tail (a full rewrite of the
        row per session per step was most of the step's host-side Python time)."""
        n = len(self.cache.pages)
        if self._bt_len < 0 or n < self._bt_len:
            self._sync_block_table()
        elif n > self._bt_len:
            self.runtime.block_table[self.seq, self._bt_len:n] = self.cache.pages[self._bt_len:n]
            self._bt_len = n


def new_session(base: BaseWeights, adapter: Optional[AdapterSet] = None, max_context: int = 512,
                ledger: Optional[Ledger] = None, runtime=None,
                capture_logits: bool = False) -> GenerationSession:
    return GenerationSession(base, adapter, max_context, ledger, runtime, capture_logits)


def _check_tokens(session: GenerationSession, tokens) -> list[int]:
    toks = [int(t) for t in tokens]
    vocab = session.config.vocab_size
    for t in toks:
        if not (0 <= t < vocab):
            raise IndexError(f"token {t} outside vocab [0, {vocab})")
    return toks


def _reads_per_step(session) -> int:
    # 7 projections per layer (wk, wv, wq, wo, gate, up, down) + the LM head (ledger
    # arithmetic of src/engine.py:166-176 with base_linear counting at model.py:334-336)
    return 7 * session.config.num_layers + 1


def _logits_np(lg, row: int) -> Optional[np.ndarray]:
    return None if lg is None else lg[row].float().cpu().numpy()


def prefill(session: GenerationSession, prompt, pool=None, namespace: Optional[str] = None,
            reader: Optional[str] = None) -> int:
    """Encode the prompt, reuse the pooled prefix, emit the first (base) token."""
    if session._prefilled:
        raise StateError("session already prefilled")
    toks = _check_tokens(session, prompt)
    if not toks:
        raise ValueError("prompt must contain at least one token")
    if len(toks) > session.max_context:
        raise CapacityError(f"prompt length {len(toks)} exceeds max context {session.max_context}")
    cfg, rt, led = session.config, session.runtime, session.ledger
    matched, chain = 0, []
    if pool is not None:
        matched, chain = pool.lookup(namespace, toks, reader=reader)
        if chain:
            if any(b.arena is not rt.arena for b in chain):
                pool.release(chain)
                raise ContractViolationError("pooled blocks live in another page arena")
            session.cache.attach_shared([b.page for b in chain])
            session.borrowed_chain = chain
        led.prefix_hit_tokens += matched

    n = len(toks)
    suffix = toks[matched:]
    if suffix:
        session.cache.ensure_pages(n - 1)
        session._sync_block_table()
        step = rt.max_rows
        token = None
        for c0 in range(matched, n, step):
            c1 = min(n, c0 + step)
            pos = np.arange(c0, c1, dtype=np.int32)
            emit = ((pos % BLOCK_TOKENS) == BLOCK_TOKENS - 1) | (pos == n - 1)
            out, lg = rt.forward(tokens=toks[c0:c1], kind=np.zeros(c1 - c0, np.int32),
                                 seq=np.full(c1 - c0, session.seq, np.int32), pos=pos,
                                 adapter=np.full(c1 - c0, -1, np.int32), emit=emit.astype(np.int32),
                                 logits=session.capture_logits and c1 == n)
            session.cache.advance(c1 - c0)
            for p, t in zip(pos[emit], out):
                session.base_next[int(p)] = int(t)
            if c1 == n:
                token = int(out[-1])
                session._set_logits(lg, int(emit.sum()) - 1, 0)
        led.prefill_tokens += len(suffix)
        led.kv_bytes_written += len(suffix) * cfg.kv_bytes_per_token
        led.param_matrix_reads += _reads_per_step(session)
        session._note_computed(matched, n)
    else:
        token = _full_hit_token(session, toks, chain)
    session.prompt = toks
    session.produced = [token]
    session._prefilled = True
    return token


def _full_hit_token(session: GenerationSession, toks: list, chain: list) -> int:
    """The whole prompt was pooled: emit the stored chunk-end prediction, or replay the last
    position through a read-only (decoder-kind, no adapter) row -- it cannot write KV
    (src/engine.py:135-148)."""
    stored = chain[-1].next_token if chain else None
    if stored is not None:
        session.last_logits = None
        return int(stored)
    n = len(toks)
    session._sync_block_table()
    out, lg = session.runtime.forward(tokens=[toks[-1]], kind=[1], seq=[session.seq], pos=[n - 1],
                                      adapter=[-1], emit=[1], logits=session.capture_logits)
    token = int(out[0])
    session.base_next[n - 1] = token
    session._set_logits(lg, 0, 1)
    session.ledger.prefill_tokens += 1
    session.ledger.param_matrix_reads += 5 * session.config.num_layers + 1
    return token


def _prefill_setup(sessions, prompts, pool, namespace, readers, rt):
    """prefill_batch's per-session part: checks, pool lookup + page attach, page mapping and
    ledger; returns the suffix rows (session index, token, position, emit) and the first
    tokens of fully pooled prompts."""
    readers = list(readers) if readers is not None else [None] * len(sessions)
    # one namespace for all, or one per session (the reference's baseline mode serves each
    # agent from its own namespace, src/simulate.py:313)
    spaces = list(namespace) if isinstance(namespace, (list, tuple)) else [namespace] * len(sessions)
    firsts: list = [None] * len(sessions)
    rows = []
    for i, (session, prompt) in enumerate(zip(sessions, prompts)):
        toks = _check_tokens(session, prompt)
        if session._prefilled:
            raise StateError("session already prefilled")
        if not toks:
            raise ValueError("prompt must contain at least one token")
        if len(toks) > session.max_context:
            raise CapacityError(f"prompt length {len(toks)} exceeds max context {session.max_context}")
        matched, chain = 0, []
        if pool is not None:
            matched, chain = pool.lookup(spaces[i], toks, reader=readers[i])
            if chain:
                if any(b.arena is not rt.arena for b in chain):
                    pool.release(chain)
                    raise ContractViolationError("pooled blocks live in another page arena")
                session.cache.attach_shared([b.page for b in chain])
                session.borrowed_chain = chain
            session.ledger.prefix_hit_tokens += matched
        n = len(toks)
        session.prompt = toks
        if matched == n:  # the whole prompt was pooled
            firsts[i] = _full_hit_token(session, toks, chain)
            continue
        session.cache.ensure_pages(n - 1)
        session._sync_block_table()
        for p in range(matched, n):
            rows.append((i, toks[p], p, p % BLOCK_TOKENS == BLOCK_TOKENS - 1 or p == n - 1))
        session.ledger.prefill_tokens += n - matched
        session.ledger.kv_bytes_written += (n - matched) * session.config.kv_bytes_per_token
        session.ledger.param_matrix_reads += _reads_per_step(session)
        session._note_computed(matched, n)
    return rows, firsts


def _collect_prefill_outputs(sessions, chunk, r0, last_row, want, out, lg, e, firsts):
    """Record one forward's results for its prefill rows (emitted outputs start at out[e])."""
    counts = {}
    for j, r in enumerate(chunk):
        counts[r[0]] = counts.get(r[0], 0) + 1
        if not r[3]:
            continue
        session = sessions[r[0]]
        session.base_next[r[2]] = int(out[e])
        if last_row[r[0]] == r0 + j:
            firsts[r[0]] = int(out[e])
            session._set_logits(lg if want[j] else None, e, 0)
        e += 1
    for i, c in counts.items():
        sessions[i].cache.advance(c)


def _finish_prefill(sessions, firsts):
    for i, session in enumerate(sessions):
        if not session._prefilled:
            session.produced = [firsts[i]]
            session._prefilled = True


def prefill_batch(sessions: Sequence[GenerationSession], prompts, pool=None,
                  namespace: Optional[str] = None, readers: Optional[Sequence] = None) -> list[int]:
    """`prefill` for many sessions at once: each session's pool lookup, then the uncached
    suffixes of all of them as encoder rows of shared forwards (max_rows rows each), so a
    batch of new turns streams the base weights once per forward instead of once per session.
    Per session the tokens, KV bytes, ledger and stored chunk-end predictions equal those of
    `prefill` (a row's result does not depend on the rows it shares a forward with)."""
    if len(prompts) != len(sessions):
        raise ValueError("one prompt per session")
    if not sessions:
        return []
    rt = sessions[0].runtime
    if any(s.runtime is not rt for s in sessions):
        raise ConfigError("sessions in one batch must share a runtime")
    if len({s.seq for s in sessions}) != len(sessions):
        raise StateError("a session appears twice in one batch")
    rows, firsts = _prefill_setup(sessions, prompts, pool, namespace, readers, rt)
    last_row = {}
    for k, r in enumerate(rows):
        last_row[r[0]] = k
    for c0 in range(0, len(rows), rt.max_rows):
        chunk = rows[c0:c0 + rt.max_rows]
        want = [sessions[r[0]].capture_logits and last_row[r[0]] == c0 + j for j, r in enumerate(chunk)]
        out, lg = rt.forward(tokens=[r[1] for r in chunk], kind=[0] * len(chunk),
                             seq=[sessions[r[0]].seq for r in chunk], pos=[r[2] for r in chunk],
                             adapter=[-1] * len(chunk), emit=[int(r[3]) for r in chunk], logits=any(want))
        _collect_prefill_outputs(sessions, chunk, c0, last_row, want, out, lg, 0, firsts)
    _finish_prefill(sessions, firsts)
    return firsts


def _pre_step(session: GenerationSession, token: int) -> int:
    if session._closed:
        raise StateError("session is closed")
    if not session._prefilled:
        raise StateError("decode before prefill")
    t = int(token)
    if not 0 <= t < session.config.vocab_size:
        raise IndexError(f"token {t} outside vocab [0, {session.config.vocab_size})")
    pos = session.cache.position_count
    if pos + 1 > session.max_context:
        raise CapacityError(f"context full at {pos}/{session.max_context}")
    return pos


def _account_step(session: GenerationSession, pos: int, passes: int, reads: int) -> None:
    """src/engine.py:166-176."""
    led, cfg = session.ledger, session.config
    led.decode_steps += 1
    led.param_passes += passes
    led.param_matrix_reads += reads
    led.kv_read_events += 1
    led.kv_bytes_read += (pos + 1) * cfg.kv_bytes_per_token
    led.kv_bytes_written += cfg.kv_bytes_per_token


def _prepare_write(session: GenerationSession, pos: int) -> None:
    session.cache.ensure_pages(pos)
    page = session.cache.pages[pos // BLOCK_TOKENS]
    if session.runtime.arena.refcount(page) != 1:
        raise ContractViolationError(f"position {pos} would be written into shared page {page}")
    session._sync_appended_pages()


def _finish_step(s: GenerationSession, p: int, out, lg, enc: int, dec: int) -> None:
    s.cache.advance(1)
    s.base_next[p] = int(out[enc])
    s._set_logits(lg, dec, 1 if dec != enc else 0)
    s._note_computed(p, p + 1)
    _account_step(s, p, passes=1, reads=_reads_per_step(s))


def decode_step_batch(sessions: Sequence[GenerationSession], tokens: Sequence[int]) -> list[int]:
    """ONE fused forward for many sessions (each its own adapter): per session an encoder
    row and -- if adapted -- a decoder row. Returns each session's next token."""
    if len(sessions) != len(tokens):
        raise ValueError("one token per session")
    if not sessions:
        return []
    rt = sessions[0].runtime
    if any(s.runtime is not rt for s in sessions):
        raise ConfigError("sessions in one batch must share a runtime")
    if len({s.seq for s in sessions}) != len(sessions):
        raise StateError("a session appears twice in one batch")
    tok, kind, seq, pos, ad, emit = [], [], [], [], [], []
    plan = []
    for s, t in zip(sessions, tokens):
        p = _pre_step(s, int(t))
        _prepare_write(s, p)
        enc = len(tok)
        tok.append(int(t)); kind.append(0); seq.append(s.seq); pos.append(p); ad.append(-1); emit.append(1)
        dec = enc
        if s.adapter is not None:
            dec = len(tok)
            tok.append(int(t)); kind.append(1); seq.append(s.seq); pos.append(p)
            ad.append(s.adapter_slot); emit.append(1)
        plan.append((s, p, enc, dec))
    want_logits = any(s.capture_logits for s in sessions)
    out, lg = rt.forward(tok, kind, seq, pos, ad, emit, logits=want_logits)
    nxt = []
    for s, p, enc, dec in plan:
        _finish_step(s, p, out, lg, enc, dec)
        nxt.append(int(out[dec]))
    return nxt


def step_batch(sessions: Sequence[GenerationSession], tokens: Sequence[int],
               new_sessions: Sequence[GenerationSession] = (), prompts=(), pool=None,
               namespace: Optional[str] = None, readers: Optional[Sequence] = None):
    """One decode step for `sessions` fused with the prefill of `new_sessions` (continuous
    batching with piggybacked prefill): the decode rows and the first prefill suffix rows
    share one forward (further prefill rows follow in max_rows forwards). Returns (next token
    per decoding session, first token per new session); each equals what decode_step_batch
    and prefill_batch return separately, bitwise."""
    if len(sessions) != len(tokens) or len(new_sessions) != len(prompts):
        raise ValueError("one token per session and one prompt per new session")
    everyone = list(sessions) + list(new_sessions)
    if not everyone:
        return [], []
    if not new_sessions:
        return decode_step_batch(sessions, tokens), []
    if not sessions:
        return [], prefill_batch(new_sessions, prompts, pool=pool, namespace=namespace, readers=readers)
    rt = everyone[0].runtime
    if any(s.runtime is not rt for s in everyone):
        raise ConfigError("sessions in one batch must share a runtime")
    if len({s.seq for s in everyone}) != len(everyone):
        raise StateError("a session appears twice in one batch")
    # decode rows (as decode_step_batch)
    tok, kind, seq, pos, ad, emit = [], [], [], [], [], []
    plan = []
    for s, t in zip(sessions, tokens):
        p = _pre_step(s, int(t))
        _prepare_write(s, p)
        enc = len(tok)
        tok.append(int(t)); kind.append(0); seq.append(s.seq); pos.append(p); ad.append(-1); emit.append(1)
        dec = enc
        if s.adapter is not None:
            dec = len(tok)
            tok.append(int(t)); kind.append(1); seq.append(s.seq); pos.append(p)
            ad.append(s.adapter_slot); emit.append(1)
        plan.append((s, p, enc, dec))
    n_dec = len(tok)
    if n_dec > rt.max_rows:
        raise CapacityError(f"{n_dec} decode rows exceed max_rows {rt.max_rows}")
    # prefill rows (as prefill_batch)
    rows, firsts = _prefill_setup(new_sessions, prompts, pool, namespace, readers, rt)
    last_row = {}
    for k, r in enumerate(rows):
        last_row[r[0]] = k
    first_take = rt.max_rows - n_dec
    spans = [(0, min(first_take, len(rows)))]
    spans += [(c0, min(c0 + rt.max_rows, len(rows))) for c0 in range(first_take, len(rows), rt.max_rows)]
    nxt = []
    for ci, (r0, r1) in enumerate(spans):
        chunk = rows[r0:r1]
        want = [new_sessions[r[0]].capture_logits and last_row[r[0]] == r0 + j for j, r in enumerate(chunk)]
        head = (tok, kind, seq, pos, ad, emit) if ci == 0 else ([], [], [], [], [], [])
        if not chunk and ci > 0:
            continue
        out, lg = rt.forward(tokens=head[0] + [r[1] for r in chunk], kind=head[1] + [0] * len(chunk),
                             seq=head[2] + [new_sessions[r[0]].seq for r in chunk],
                             pos=head[3] + [r[2] for r in chunk], adapter=head[4] + [-1] * len(chunk),
                             emit=head[5] + [int(r[3]) for r in chunk],
                             logits=any(want) or (ci == 0 and any(s.capture_logits for s in sessions)))
        e = 0
        if ci == 0:
            for s, p, enc, dec in plan:
                _finish_step(s, p, out, lg, enc, dec)
                nxt.append(int(out[dec]))
            e = n_dec  # every decode row emits
        _collect_prefill_outputs(new_sessions, chunk, r0, last_row, want, out, lg, e, firsts)
    _finish_prefill(new_sessions, firsts)
    return nxt, firsts


def decode_step_fused(session: GenerationSession, token: int) -> int:
    """One fused pair step (engine.py:179-193): a batch of one session."""
    return decode_step_batch([session], [token])[0]


def decode_step_sequential(session: GenerationSession, token: int) -> int:
    """Oracle-shaped path (engine.py:196-215): an encoder pass that writes K/V, then a
    read-only decoder pass -- two parameter sweeps. Same kernels, two forwards."""
    pos = _pre_step(session, token)
    _prepare_write(session, pos)
    rt = session.runtime
    out, _ = rt.forward([token], [0], [session.seq], [pos], [-1], [1])
    session.cache.advance(1)
    session.base_next[pos] = int(out[0])
    session._note_computed(pos, pos + 1)
    out2, lg = rt.forward([token], [1], [session.seq], [pos], [session.adapter_slot], [1],
                          logits=session.capture_logits)
    session._set_logits(lg, 0, 1)
    L = session.config.num_layers
    _account_step(session, pos, passes=2, reads=7 * L + 5 * L + 1)
    return int(out2[0])


def decode_step_base(session: GenerationSession, token: int) -> int:
    """Bare-base step (engine.py:218-233); refuses adapted sessions."""
    if session.adapter is not None:
        raise StateError("base decode on a session that carries an adapter")
    return decode_step_batch([session], [token])[0]


_STEPS = {"fused": decode_step_fused, "sequential": decode_step_sequential}


def generate(session: GenerationSession, prompt, max_new: int, path: str = "fused", pool=None,
             namespace: Optional[str] = None, reader: Optional[str] = None,
             end_token: Optional[int] = None) -> list[int]:
    """Prefill then greedy-decode up to max_new tokens, first one included (engine.py:239-252)."""
    if max_new < 1:
        raise ValueError(f"max_new must be at least 1, got {max_new}")
    if path not in _STEPS:
        raise ModeError(f"decode path must be one of {sorted(_STEPS)}, got {path!r}")
    step = _STEPS[path]
    out = [prefill(session, prompt, pool=pool, namespace=namespace, reader=reader)]
    while len(out) < max_new and out[-1] != end_token:
        out.append(step(session, out[-1]))
    session.produced = list(out)
    return out


def generate_batch(sessions: Sequence[GenerationSession], prompts, max_new: int, pool=None,
                   namespace: Optional[str] = None, readers=None,
                   end_token: Optional[int] = None) -> list[list[int]]:
    """B200 extension: prefill each session (pool-aware, in order, so later sessions hit
    the prefix earlier ones committed) then advance all of them with batched fused steps."""
    readers = readers or [None] * len(sessions)
    outs = [[prefill(s, p, pool=pool, namespace=namespace, reader=r)]
            for s, p, r in zip(sessions, prompts, readers)]
    live = [i for i in range(len(sessions)) if max_new > 1 and outs[i][-1] != end_token]
    while live:
        nxt = decode_step_batch([sessions[i] for i in live], [outs[i][-1] for i in live])
        for i, t in zip(live, nxt):
            outs[i].append(t)
        live = [i for i in live if len(outs[i]) < max_new and outs[i][-1] != end_token]
    for s, o in zip(sessions, outs):
        s.produced = list(o)
    return outs


def replay_base(base: BaseWeights, tokens, prompt_len: int, max_context: Optional[int] = None,
                ledger: Optional[Ledger] = None, runtime=None) -> GenerationSession:
    """Force the bare base model over a fixed token sequence (engine.py:255-271)."""
    toks = [int(t) for t in tokens]
    if not (1 <= prompt_len <= len(toks)):
        raise ValueError(f"prompt_len {prompt_len} outside [1, {len(toks)}]")
    session = new_session(base, None, max_context or len(toks) + 1, ledger, runtime)
    prefill(session, toks[:prompt_len])
    for t in toks[prompt_len:]:
        decode_step_base(session, t)
    return session


def base_next_token_at(session: GenerationSession, pos: int) -> int:
    """Greedy base prediction at a position this session computed (engine.py:274-284):
    StateError for positions it did not compute (pooled prefix, a stored full hit)."""
    if not session.computed(pos):
        raise StateError(f"position {pos} was not computed by this session")
    tok = session.base_next.get(pos)
    if tok is None:
        # Not emitted during prefill: a read-only row at `pos` reproduces the encoder row's
        # prediction bit for bit (row-independent kernels, same keys 0..pos). Emit flag 2:
        # it does not replace the hidden state kept for last_logits.
        session._sync_block_table()
        fed = session.prompt + session.produced
        out, _ = session.runtime.forward([fed[pos]], [1], [session.seq], [pos], [-1], [2])
        tok = int(out[0])
        session.base_next[pos] = tok
    session.ledger.param_matrix_reads += 1
    return tok
