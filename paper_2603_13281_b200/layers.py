"""The reference's module-level model functions on the B200 kernels.

Drop-in for src/model.py:334-538 -- `base_linear`, `adapted_linear`, `icarus_linear`
(:334-371), `causal_mask`, `layer_attention` (:378-425), `block_forward` (:441-508) and
`decoder_block_readonly` (:511-538) -- with the same signatures, argument meaning, guards and
exception classes, re-exported from `paper_2603_13281_b200.model`. Every computation runs
through the C ABI on the device; there is no CPU path:

  base_linear / adapted_linear / icarus_linear  -> icr_linear_bf16: the tcgen05 stream-K
      projection GEMM with the LoRA shrink + expand inside it, as in the decode step. The
      low-rank chunk is always part of the launch (zero U on rows without an adapter), so a
      row's bits do not depend on whether an adapter rides along: base_linear ==
      adapted_linear with B = 0 == icarus_linear's encoder row, bitwise (the reference's
      tests/test_model.py:106-132).
  layer_attention -> icr_paged_attention: the shared-KV paged attention kernel over pages
      built from the given K/V rows; a 2H-head query row is the pair (encoder heads, decoder
      heads) of the fused step, exactly how the engine feeds it.
  block_forward / decoder_block_readonly -> icr_layer_forward: one layer of the fused
      forward (the same kernels, same order) over explicit fp32 rows, with the session cache's
      pages as block-table row; encoder rows append K/V to that layer.

Values are bf16 operands with fp32 accumulation (the product precision), so results match the
reference within the bf16 tolerance the GPU tests state, not bitwise; the structural
identities above are bitwise.
"""

from __future__ import annotations

import numpy as np

from .errors import (ConfigError, ContractViolationError, DeviceError, ModeError, ShapeError,
                     StateError)
from .model import BLOCK_TOKENS, Param

NEG_MASK = -1e30  # src/tensor.py:31-33
MAX_RANK = 32     # the kernels' LoRA rank bound (runtime.cu: lora_rank <= 32)


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
    return torch


def _arr(x) -> np.ndarray:
    """The array behind a reference Tensor / Param / ndarray argument."""
    data = getattr(x, "data", x)
    if hasattr(data, "detach"):
        return data.detach().float().cpu().numpy()
    return np.asarray(data)


def _lib():
    from . import _lib as L
    return L, L.load()


def _pad_to(n: int, m: int) -> int:
    return (n + m - 1) // m * m


# ----------------------------------------------------------------------------- weights
_WCACHE: dict = {}  # id(weight) -> (weight, device [M, K] bf16); the weight ref keeps id stable
_WCACHE_MAX = 64


def _device_weight(w):
    """W [in, out] (reference layout) -> device bf16 [out_pad, in_pad] (K-major), cached."""
    torch = _torch()
    key = id(w)
    hit = _WCACHE.get(key)
    if hit is not None and hit[0] is w:
        return hit[1]
    a = _arr(w)
    if a.ndim != 2:
        raise ShapeError(f"weight must be 2-D, got {a.shape}")
    k_in, out = a.shape
    dev = torch.zeros(_pad_to(out, 128), _pad_to(k_in, 64), dtype=torch.bfloat16, device="cuda")
    dev[:out, :k_in] = torch.from_numpy(np.ascontiguousarray(a.T, dtype=np.float32)).to("cuda")
    if len(_WCACHE) >= _WCACHE_MAX:
        _WCACHE.pop(next(iter(_WCACHE)))
    _WCACHE[key] = (w, dev)
    return dev


def _lowrank_operands(pair, scaling: float, k_pad: int, m_pad: int):
    """A [r, in] -> bf16 [r, K]; scaling * B [out, r] -> bf16 tile-major [M/128][1][128][64]."""
    from .runtime import tile_major
    torch = _torch()
    a, b = _arr(pair.a), _arr(pair.b)
    r = a.shape[0]
    if r < 1 or r > MAX_RANK:
        raise ConfigError(f"B200 low-rank term supports rank 1..{MAX_RANK}, got {r}")
    ad = torch.zeros(r, k_pad, dtype=torch.bfloat16, device="cuda")
    ad[:, :a.shape[1]] = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to("cuda")
    bs = torch.zeros(m_pad, 64, dtype=torch.float32, device="cuda")
    bs[:b.shape[0], :r] = torch.from_numpy(np.ascontiguousarray(b, dtype=np.float32)).to("cuda") * float(scaling)
    return ad, tile_major(bs.to(torch.bfloat16)), r


def _linear(x, w, pair, scaling: float, adapted_rows) -> Param:
    torch = _torch()
    L, lib = _lib()
    xa = _arr(x)
    if xa.ndim != 2:
        raise ShapeError(f"linear input must be 2-D, got {xa.shape}")
    wd = _device_weight(w)
    k_in, out = _arr(w).shape
    if xa.shape[1] != k_in:
        raise ShapeError(f"cannot multiply {xa.shape} by {(k_in, out)}")
    M, K = wd.shape
    n = xa.shape[0]
    xd = torch.zeros(n, K, dtype=torch.bfloat16, device="cuda")
    xd[:, :k_in] = torch.from_numpy(np.ascontiguousarray(xa, dtype=np.float32)).to("cuda")
    y = torch.empty(n, M, dtype=torch.float32, device="cuda")
    if pair is not None:
        ad, bsd, r = _lowrank_operands(pair, scaling, K, M)
        flags = np.ascontiguousarray(adapted_rows, dtype=np.int32)
        L.check(lib.icr_linear_bf16(wd.data_ptr(), xd.data_ptr(), y.data_ptr(), M, K, n,
                                    ad.data_ptr(), bsd.data_ptr(), r, L.i32_ptr(flags),
                                    L.stream_handle()))
    else:
        L.check(lib.icr_linear_bf16(wd.data_ptr(), xd.data_ptr(), y.data_ptr(), M, K, n,
                                    None, None, 0, None, L.stream_handle()))
    return Param(y[:, :out].cpu().numpy())


def base_linear(x, w, ledger=None) -> Param:
    """src/model.py:334-337: x @ W, one parameter-read event."""
    if ledger is not None:
        ledger.param_matrix_reads += 1
    return _linear(x, w, None, 0.0, None)


def adapted_linear(x, w, pair, scaling: float, ledger=None) -> Param:
    """src/model.py:346-352: base projection plus the low-rank term on every row."""
    if ledger is not None:
        ledger.param_matrix_reads += 1
    n = _arr(x).shape[0]
    return _linear(x, w, pair, scaling, np.ones(n, np.int32))


def icarus_linear(x_pair, w, pair, scaling: float, ledger=None) -> Param:
    """src/model.py:355-371: one weight pass for the [2, in] pair, the low-rank term on row 1
    (the decoder branch) only."""
    xa = _arr(x_pair)
    if xa.ndim != 2 or xa.shape[0] != 2:
        raise ShapeError(f"icarus_linear needs a [2, in_dim] pair, got {xa.shape}")
    if ledger is not None:
        ledger.param_matrix_reads += 1
    return _linear(xa, w, pair, scaling, np.array([0, 1], np.int32))


# ----------------------------------------------------------------------------- attention
def causal_mask(query_positions, key_count: int, dtype=np.float32) -> Param:
    """src/model.py:378-381: additive NEG_MASK where the key index exceeds the query
    position (host metadata; the attention kernel applies the same rule in-kernel)."""
    qp = np.atleast_1d(np.asarray(query_positions, dtype=np.int64))
    dt = np.dtype(dtype)
    bad = np.arange(key_count)[None, :] > qp[:, None]
    return Param(np.where(bad, dt.type(NEG_MASK), dt.type(0.0)))


def layer_attention(q, k, v, query_positions, config) -> Param:
    """src/model.py:384-425: GQA over H or 2H query heads (heads H..2H-1 are the decoder
    branch and reuse the groups of head h mod H), on the shared-KV paged attention kernel."""
    from .runtime import auto_chunk_pages
    qa, ka, va = _arr(q), _arr(k), _arr(v)
    dk, H, Hkv = config.head_dim, config.num_heads, config.num_kv_heads
    if qa.ndim != 2 or qa.shape[1] % dk != 0:
        raise ShapeError(f"q shape {qa.shape} is not a multiple of head_dim {dk}")
    n_heads = qa.shape[1] // dk
    if n_heads not in (H, 2 * H):
        raise ModeError(f"query head count {n_heads} must be {H} or {2 * H}")
    if ka.shape != va.shape or ka.ndim != 2 or ka.shape[1] != config.kv_dim:
        raise ShapeError(f"k/v shapes {ka.shape}/{va.shape} do not match kv_dim {config.kv_dim}")
    T = ka.shape[0]
    if T < 1:
        raise StateError("attention over an empty cache")
    qpos = np.atleast_1d(np.asarray(query_positions, dtype=np.int64))
    if qpos.shape[0] != qa.shape[0]:
        raise ShapeError(f"{qpos.shape[0]} query positions for {qa.shape[0]} rows")
    if qpos.max() >= T:
        raise StateError(f"query position {qpos.max()} has no key (cache length {T})")
    torch = _torch()
    L, lib = _lib()
    S = qa.shape[0]
    rep = n_heads // H  # a 2H row = (encoder heads, decoder heads): two kernel rows
    rows = S * rep
    qd = torch.from_numpy(np.ascontiguousarray(qa, dtype=np.float32)).to("cuda", torch.bfloat16)
    qd = qd.reshape(rows, H * dk).contiguous()
    P = -(-T // BLOCK_TOKENS)

    def pages(x):
        buf = torch.zeros(P * BLOCK_TOKENS, Hkv, dk, dtype=torch.bfloat16, device="cuda")
        buf[:T] = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to("cuda").view(T, Hkv, dk)
        return buf.view(P, BLOCK_TOKENS, Hkv, dk).permute(0, 2, 1, 3).contiguous()

    kp, vp = pages(ka), pages(va)
    row_seq = np.zeros(rows, np.int32)
    row_pos = np.ascontiguousarray(np.repeat(qpos, rep), dtype=np.int32)
    bt = np.arange(P, dtype=np.int32)
    out = torch.empty(rows, H * dk, dtype=torch.bfloat16, device="cuda")
    n_items = np.zeros(1, np.int32)
    L.check(lib.icr_paged_attention(qd.data_ptr(), kp.data_ptr(), vp.data_ptr(), H, Hkv, dk,
                                    auto_chunk_pages(T), rows, L.i32_ptr(row_seq),
                                    L.i32_ptr(row_pos), L.i32_ptr(bt), 1, P, out.data_ptr(),
                                    L.i32_ptr(n_items), L.stream_handle()))
    return Param(out.float().reshape(S, n_heads * dk).cpu().numpy())


# ----------------------------------------------------------------------------- blocks
def _layer_call(base, adapter, cache, layer: int, x: np.ndarray, kind, pos, writes: bool):
    """Run rows through layer `layer` of the device forward with the cache's pages."""
    torch = _torch()
    rt = base.runtime()
    if cache.arena is not rt.arena:
        raise ContractViolationError(
            "the cache's pages must live in the runtime's page arena: create it with "
            "KvCacheTensor(config, capacity, arena=base.runtime().arena)")
    slot = rt.slots.slot_of(adapter) if adapter is not None else -1
    n = x.shape[0]
    if writes:
        last = int(max(pos))
        if last >= cache.capacity:
            from .errors import CapacityError
            raise CapacityError(f"cache layer {layer} at {cache.length(layer)}/{cache.capacity} "
                                f"cannot take {n} more positions")
        cache.ensure_pages(last)
        for p in sorted({int(p) // BLOCK_TOKENS for p in pos}):
            if rt.arena.refcount(cache.pages[p]) > 1:
                raise ContractViolationError(f"append into shared page {cache.pages[p]}")
    seq = rt.acquire_seq()
    try:
        rt.set_pages(seq, cache.pages)
        xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to("cuda")
        kind = np.asarray(kind, np.int32)
        pos = np.asarray(pos, np.int32)
        ad = np.where(kind == 1, slot, -1).astype(np.int32)
        outs = []
        for c0 in range(0, n, rt.max_rows):
            c1 = min(n, c0 + rt.max_rows)
            outs.append(rt.layer_forward(xd[c0:c1], layer, kind[c0:c1], np.full(c1 - c0, seq, np.int32),
                                         pos[c0:c1], ad[c0:c1]))
            if writes:
                cache.advance_layer(layer, int((kind[c0:c1] == 0).sum()))
    finally:
        rt.release_seq(seq)
    return Param(torch.cat(outs).cpu().numpy())


def block_forward(x, layer: int, base, adapter, cache, mode: str, positions, ledger=None) -> Param:
    """src/model.py:441-508: one layer, batched base-only prefill ([S, d], adapters ignored,
    S new cache positions) or the fused pair decode ([2, d]; K/V from row 0, appended before
    attention so both branches see the current position)."""
    cfg = base.config
    xa = _arr(x)
    pos = np.atleast_1d(np.asarray(positions, dtype=np.int64))
    if cache.length(layer) != pos[0]:
        raise StateError(f"layer {layer} cache length {cache.length(layer)} "
                         f"does not match first position {pos[0]}")
    if xa.ndim != 2 or xa.shape[1] != cfg.hidden_dim:
        raise ShapeError(f"block input must be [rows, {cfg.hidden_dim}], got {xa.shape}")
    if mode == "prefill":
        if pos.shape[0] != xa.shape[0]:
            raise ShapeError(f"{pos.shape[0]} positions for {xa.shape[0]} rows")
        out = _layer_call(base, None, cache, layer, xa, np.zeros(len(pos), np.int32), pos, True)
    elif mode == "decode":
        if xa.shape[0] != 2:
            raise ShapeError(f"decode mode expects a [2, hidden] pair, got {xa.shape}")
        if pos.shape[0] != 1:
            raise ShapeError(f"decode mode takes one position, got {pos.shape[0]}")
        out = _layer_call(base, adapter, cache, layer, xa, np.array([0, 1], np.int32),
                          np.repeat(pos, 2), True)
    else:
        raise ModeError(f"block mode must be prefill or decode, got {mode!r}")
    if ledger is not None:
        ledger.param_matrix_reads += 7  # wk, wv, wq, wo, gate, up, down
    return out


def decoder_block_readonly(x, layer: int, base, adapter, cache, position: int,
                           ledger=None) -> Param:
    """src/model.py:511-538: the decoder pass of the sequential decode over a cache that
    already holds `position`; never writes the cache (a decoder-kind row)."""
    cfg = base.config
    if cache.length(layer) != position + 1:
        raise StateError(f"readonly decode at position {position} needs cache length "
                         f"{position + 1}, layer {layer} has {cache.length(layer)}")
    xa = _arr(x)
    if xa.ndim != 2 or xa.shape != (1, cfg.hidden_dim):
        raise ShapeError(f"readonly decode expects [1, {cfg.hidden_dim}], got {xa.shape}")
    out = _layer_call(base, adapter, cache, layer, xa, np.array([1], np.int32),
                      np.array([position]), False)
    if ledger is not None:
        ledger.param_matrix_reads += 5  # wq, wo, gate, up, down
    return out


__all__ = ["base_linear", "adapted_linear", "icarus_linear", "causal_mask", "layer_attention",
           "block_forward", "decoder_block_readonly"]
