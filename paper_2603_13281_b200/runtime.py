"""Device residency and the bridge to the sm_100a library.

  PageArena      the shared KV page store: K and V arenas [L, pages, H_kv, 16, hd] bf16,
                 a free list and per-page reference counts. One page = one pool block
                 (BLOCK_TOKENS = 16 positions) for all layers.
  DeviceWeights  the base model packed for the kernels: bf16, [out, in] (K-major),
                 RMSNorm gains folded into the following projection, wq|wk|wv fused,
                 gate/up rows interleaved, LM head padded to a multiple of 128 rows.
  AdapterSlots   resident LoRA adapters (reference A as-is, B pre-multiplied by
                 alpha/rank), addressed by slot; the decode step picks a slot per row.
  Runtime        owns the above plus the C model handle and the host block table;
                 `forward` is one fused multi-model step (icr_forward).

Memory is allocated with torch (plumbing); all compute is the library's CUDA kernels.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from typing import Optional

import numpy as np

from . import _lib
from .errors import CapacityError, ConfigError, ContractViolationError, DeviceError
from .model import BLOCK_TOKENS, DECODER_TARGETS, AdapterSet, ModelConfig


def _torch():
    import torch
    return torch


# ----------------------------------------------------------------------------- pages
class PageArena:
    """Reference-counted 16-token KV pages shared by sessions and the prefix pool."""

    def __init__(self, config: ModelConfig, num_pages: int, device="cuda"):
        torch = _torch()
        if num_pages < 1:
            raise ConfigError(f"page arena needs at least one page, got {num_pages}")
        self.config = config
        self.num_pages = num_pages
        shape = (config.num_layers, num_pages, config.num_kv_heads, BLOCK_TOKENS, config.head_dim)
        self.k = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.v = torch.zeros(shape, dtype=torch.bfloat16, device=device)
        self.refs = np.zeros(num_pages, dtype=np.int32)
        self.gen = np.zeros(num_pages, dtype=np.int64)  # bumped per allocation: page identity
        self._free = list(range(num_pages - 1, -1, -1))
        self._reclaimers: list = []  # weak refs to prefix pools holding pages of this arena

    @classmethod
    def host_only(cls, config: ModelConfig, pages: int) -> "PageArena":
        return cls(config, max(pages, 1), device="cpu")

    @property
    def page_bytes(self) -> int:
        return self.config.num_layers * 2 * self.config.num_kv_heads * BLOCK_TOKENS * self.config.head_dim * 2

    def layer_ptrs(self, layer: int) -> tuple[int, int]:
        stride = self.k.stride(0) * self.k.element_size()
        return self.k.data_ptr() + layer * stride, self.v.data_ptr() + layer * stride

    def free_pages(self) -> int:
        return len(self._free)

    def register_reclaimer(self, pool) -> None:
        """A prefix pool that holds page references here: when the arena runs dry, its
        unpinned blocks are evicted (LRU) before allocation fails -- the device pages, not
        only the pool's byte budget, bound what the pool may keep."""
        import weakref
        if not any(r() is pool for r in self._reclaimers):
            self._reclaimers.append(weakref.ref(pool))

    def alloc(self) -> int:
        if not self._free:
            for ref in list(self._reclaimers):
                pool = ref()
                if pool is not None and not self._free:
                    pool.reclaim_pages(self, 1)
        if not self._free:
            raise CapacityError(f"KV page arena exhausted ({self.num_pages} pages)")
        pid = self._free.pop()
        self.refs[pid] = 1
        self.gen[pid] += 1
        return pid

    def incref(self, pid: int) -> None:
        if self.refs[pid] < 1:
            raise ContractViolationError(f"incref of free page {pid}")
        self.refs[pid] += 1

    def decref(self, pid: int) -> None:
        if self.refs[pid] < 1:
            raise ContractViolationError(f"double free of page {pid}")
        self.refs[pid] -= 1
        if self.refs[pid] == 0:
            self._free.append(pid)

    def refcount(self, pid: int) -> int:
        return int(self.refs[pid])

    # swap (pool eviction policy "swap", src/kvpool.py:282-356) ----------------------
    def save_page(self, pid: int):
        """Copy page pid's K/V (every layer) into host memory -- pinned, queued on the current
        stream, so a later writer of the recycled page is ordered after the copy."""
        torch = _torch()
        pin = self.k.is_cuda
        shape = (self.config.num_layers, self.config.num_kv_heads, BLOCK_TOKENS, self.config.head_dim)
        kh = torch.empty(shape, dtype=torch.bfloat16, pin_memory=pin)
        vh = torch.empty(shape, dtype=torch.bfloat16, pin_memory=pin)
        kh.copy_(self.k[:, pid], non_blocking=pin)
        vh.copy_(self.v[:, pid], non_blocking=pin)
        return kh, vh

    def load_page(self, pid: int, saved) -> None:
        """Inverse of save_page into (freshly allocated) page pid."""
        self.k[:, pid].copy_(saved[0], non_blocking=True)
        self.v[:, pid].copy_(saved[1], non_blocking=True)

    def host_rows(self, saved, layer: int):
        """[16, Hkv, hd] float K and V rows of one layer of a saved page."""
        torch = _torch()
        if self.k.is_cuda:
            torch.cuda.current_stream().synchronize()  # the D2H copy was queued asynchronously
        return (saved[0][layer].transpose(0, 1).float().numpy(),
                saved[1][layer].transpose(0, 1).float().numpy())

    # host-side row access (tests, copy-in, fingerprints) --------------------------
    def _index(self, pages, start, stop):
        pos = np.arange(start, stop)
        return (np.asarray(pages, dtype=np.int64)[pos // BLOCK_TOKENS], pos % BLOCK_TOKENS)

    def write_rows(self, layer, pages, at, k, v) -> None:
        torch = _torch()
        pid, slot = self._index(pages, at, at + k.shape[0])
        pid_t = torch.as_tensor(pid, device=self.k.device)
        slot_t = torch.as_tensor(slot, device=self.k.device)
        kt = torch.as_tensor(np.asarray(k, dtype=np.float32)).to(self.k.device, torch.bfloat16)
        vt = torch.as_tensor(np.asarray(v, dtype=np.float32)).to(self.k.device, torch.bfloat16)
        self.k[layer, pid_t, :, slot_t] = kt
        self.v[layer, pid_t, :, slot_t] = vt

    def _gather(self, layer, pages, start, stop):
        torch = _torch()
        pid, slot = self._index(pages, start, stop)
        pid_t = torch.as_tensor(pid, device=self.k.device)
        slot_t = torch.as_tensor(slot, device=self.k.device)
        return self.k[layer, pid_t, :, slot_t], self.v[layer, pid_t, :, slot_t]  # [n, Hkv, hd]

    def read_rows(self, layer, pages, start, stop):
        k, v = self._gather(layer, pages, start, stop)
        return k.float().cpu().numpy(), v.float().cpu().numpy()

    def read_raw(self, layer, pages, start, stop) -> tuple[bytes, bytes]:
        if stop <= start:
            return b"", b""
        torch = _torch()
        k, v = self._gather(layer, pages, start, stop)
        as_bytes = lambda t: t.contiguous().view(torch.int16).cpu().numpy().tobytes()  # noqa: E731
        return as_bytes(k), as_bytes(v)


# ----------------------------------------------------------------------------- weights
def tile_major(w):
    """[M, K] -> [M/128, K/64, 128, 64] contiguous: every 128x64 GEMM tile is one 16 KB
    block, so a weight-streaming CTA reads long contiguous runs of HBM (3-D TMA box)."""
    M, K = w.shape
    return w.view(M // 128, 128, K // 64, 64).permute(0, 2, 1, 3).contiguous()


def untile(w):
    """Inverse of tile_major (tests, checksums)."""
    mt, kt, _, _ = w.shape
    return w.permute(0, 2, 1, 3).reshape(mt * 128, kt * 64)


class DeviceWeights:
    """Base weights in the kernel layout (see module doc)."""

    def __init__(self, config: ModelConfig):
        self.config = config
        self.layers: list[dict] = []
        self.embed = None
        self.lm_head = None

    @property
    def vocab_pad(self) -> int:
        return (self.config.vocab_size + 127) // 128 * 128

    @classmethod
    def from_host(cls, base, device="cuda") -> "DeviceWeights":
        torch = _torch()
        cfg = base.config
        cfg.check_device_shapes()
        self = cls(cfg)
        bf = torch.bfloat16

        def t(a):
            return torch.from_numpy(np.array(a, dtype=np.float32, copy=True))

        for lw in base.layers:
            g_attn = t(lw.attn_gain.data)[None, :]
            g_ffn = t(lw.ffn_gain.data)[None, :]
            qkv = torch.cat([t(lw.wq.data).T, t(lw.wk.data).T, t(lw.wv.data).T], 0) * g_attn
            gate = t(lw.gate.data).T * g_ffn
            up = t(lw.up.data).T * g_ffn
            gu = torch.stack([gate, up], 1).reshape(2 * cfg.ffn_dim, cfg.hidden_dim)
            self.layers.append({
                "w_qkv": tile_major(qkv.to(device, bf)),
                "w_o": tile_major(t(lw.wo.data).T.contiguous().to(device, bf)),
                "w_gu": tile_major(gu.to(device, bf)),
                "w_down": tile_major(t(lw.down.data).T.contiguous().to(device, bf)),
            })
        self.embed = t(base.embed.data).to(device, bf).contiguous()
        lm = torch.zeros(self.vocab_pad, cfg.hidden_dim)
        lm[:cfg.vocab_size] = t(base.lm_head.data).T * t(base.final_gain.data)[None, :]
        self.lm_head = tile_major(lm.to(device, bf))
        return self

    @classmethod
    def random(cls, cfg: ModelConfig, seed: int, device="cuda") -> "DeviceWeights":
        torch = _torch()
        cfg.check_device_shapes()
        self = cls(cfg)
        gen = torch.Generator(device=device)
        gen.manual_seed(int(seed))
        bf = torch.bfloat16
        d, qd, kvd, f = cfg.hidden_dim, cfg.q_dim, cfg.kv_dim, cfg.ffn_dim

        def draw(rows, cols, fan_in):
            out = torch.empty(rows, cols, dtype=bf, device=device)
            step = max(1, (1 << 26) // cols)
            for r0 in range(0, rows, step):
                r1 = min(rows, r0 + step)
                out[r0:r1] = (torch.randn(r1 - r0, cols, generator=gen, device=device)
                              / math.sqrt(fan_in)).to(bf)
            return out

        for _ in range(cfg.num_layers):
            self.layers.append({
                "w_qkv": tile_major(draw(qd + 2 * kvd, d, d)), "w_o": tile_major(draw(d, qd, qd)),
                "w_gu": tile_major(draw(2 * f, d, d)), "w_down": tile_major(draw(d, f, f))})
        self.embed = draw(cfg.vocab_size, d, d)
        lm = draw(self.vocab_pad, d, d)
        lm[cfg.vocab_size:] = 0
        self.lm_head = tile_major(lm)
        return self

    def checksum(self) -> str:
        torch = _torch()
        acc = 0.0
        for lw in self.layers:
            for w in lw.values():
                acc += float(w.float().sum(dtype=torch.float64)) if w.numel() < (1 << 24) else float(
                    w[::97].float().sum(dtype=torch.float64))
        acc += float(self.embed.float().sum(dtype=torch.float64))
        return f"{acc:.10e}"

    def nbytes_streamed(self) -> int:
        """Weight bytes one decode step streams (embedding is gathered, not streamed)."""
        n = sum(w.numel() * w.element_size() for lw in self.layers for w in lw.values())
        return n + self.config.vocab_size * self.config.hidden_dim * 2


# ----------------------------------------------------------------------------- adapters
_A_KEYS = ("a_q", "a_o", "a_gate", "a_up", "a_down")


def lora_k(n_u: int, slots: int, rank: int) -> int:
    """K extent of a LoRA expand operand: n_u targets x slots x rank, padded to 64."""
    return (n_u * slots * rank + 63) // 64 * 64


class AdapterSlots:
    """Resident LoRA adapters; slot s of every tensor belongs to one AdapterSet.

    A (the shrink operand) is kept as the reference stores it: [L, slots, r, in].
    B (the expand operand) is concatenated over slots along K and stored tile-major like
    the base weights: b_* = [L, M/128, Kc/64, 128, 64] with element (m, t*S*r + s*r + j) =
    (alpha/r) * B_s,t[m, j]. The GEMM multiplies it by a block-diagonal U (row n carries
    its adapter's U in its own slot, zeros elsewhere), so the SGMV expand runs as extra
    tcgen05 K-chunks of the base projection. gate/up use two target blocks (t = 0 gate on
    even rows, t = 1 up on odd rows); q rows of w_qkv carry B_q, k/v rows are zero."""

    def __init__(self, cfg: ModelConfig, slots: int, rank: int, device="cuda"):
        torch = _torch()
        self.cfg, self.n, self.rank, self.device = cfg, slots, rank, device
        L, d, qd, kvd, f = cfg.num_layers, cfg.hidden_dim, cfg.q_dim, cfg.kv_dim, cfg.ffn_dim
        z = lambda *s: torch.zeros(*s, dtype=torch.bfloat16, device=device)  # noqa: E731
        self.t = {}
        self.b = {}
        if slots > 0 and rank > 0:
            self.t = {"a_q": z(L, slots, rank, d), "a_o": z(L, slots, rank, qd),
                      "a_gate": z(L, slots, rank, d), "a_up": z(L, slots, rank, d),
                      "a_down": z(L, slots, rank, f)}
            k1, k2 = lora_k(1, slots, rank), lora_k(2, slots, rank)
            for key, M, K in (("b_q", qd + 2 * kvd, k1), ("b_o", d, k1), ("b_gu", 2 * f, k2),
                              ("b_down", d, k1)):
                self.b[key] = z(L, M // 128, K // 64, 128, 64)
        self._owner: dict[int, int] = {}  # id(adapter) -> slot
        self._refs: list = [None] * slots

    def slot_of(self, adapter: AdapterSet) -> int:
        """The adapter's resident slot (uploaded on first use). Served adapters are treated as
        immutable: after changing an adapter's weights in place, call `release(adapter)` so
        the next use uploads the new values."""
        key = id(adapter)
        if key in self._owner:
            return self._owner[key]
        if self.n == 0 or self.rank == 0:
            raise CapacityError("runtime has no adapter slots (adapter_slots=0)")
        if adapter.rank > self.rank:
            raise ConfigError(f"adapter rank {adapter.rank} exceeds slot rank {self.rank}")
        free = [i for i, r in enumerate(self._refs) if r is None]
        if not free:
            raise CapacityError(f"all {self.n} adapter slots are in use")
        s = free[0]
        self._upload(s, adapter)
        self._owner[key] = s
        self._refs[s] = adapter
        return s

    def _put_b(self, key: str, layer: int, s: int, target: int, rows, value) -> None:
        """Write value [len(rows), r] (already scaled) as slot s / target of b_key[layer]."""
        torch = _torch()
        r = self.rank
        bt = self.b[key][layer]                           # [Mt, Kt, 128, 64]
        view = bt.permute(0, 2, 1, 3)                     # [Mt, 128, Kt, 64] logical (m, k)
        col = target * self.n * r + s * r
        Mt = bt.shape[0]
        full = torch.zeros(Mt * 128, r, dtype=torch.bfloat16, device=self.device)
        vv = value.to(self.device, torch.bfloat16)
        full[rows, :vv.shape[1]] = vv
        full = full.view(Mt, 128, r)
        # the slot's r columns may straddle a 64-column block (rank 24, slot >= 2)
        j = 0
        while j < r:
            kt, kin = (col + j) // 64, (col + j) % 64
            w = min(r - j, 64 - kin)
            view[:, :, kt, kin:kin + w] = full[:, :, j:j + w]
            j += w

    def _upload(self, s: int, ad: AdapterSet) -> None:
        torch = _torch()
        cfg = self.cfg
        for key in self.t:
            self.t[key][:, s].zero_()
        qd, f, d = cfg.q_dim, cfg.ffn_dim, cfg.hidden_dim
        rows = {"q": slice(0, qd), "o": slice(0, d), "gate": slice(0, 2 * f, 2),
                "up": slice(1, 2 * f, 2), "down": slice(0, d)}
        where = {"q": ("b_q", 0), "o": ("b_o", 0), "gate": ("b_gu", 0), "up": ("b_gu", 1),
                 "down": ("b_down", 0)}
        gen = None
        if ad.device_seed is not None:
            gen = torch.Generator(device=self.device)
            gen.manual_seed(int(ad.device_seed))
        sc = float(ad.scaling)
        fan = {"q": d, "o": qd, "gate": d, "up": d, "down": f}
        outd = {"q": qd, "o": d, "gate": f, "up": f, "down": d}
        for layer in range(cfg.num_layers):
            per = ad.layers[layer]
            for tgt in ("q", "o", "gate", "up", "down"):
                if gen is not None:
                    a = torch.randn(ad.rank, fan[tgt], generator=gen, device=self.device) / math.sqrt(fan[tgt])
                    b = torch.randn(outd[tgt], ad.rank, generator=gen, device=self.device) * ad.b_scale
                elif tgt in per:
                    a = torch.from_numpy(np.array(per[tgt].a.data, dtype=np.float32, copy=True))
                    b = torch.from_numpy(np.array(per[tgt].b.data, dtype=np.float32, copy=True))
                else:
                    continue
                self.t["a_" + tgt][layer, s, :ad.rank] = a.to(self.device, torch.bfloat16)
                key, target = where[tgt]
                self._put_b(key, layer, s, target, rows[tgt], b * sc)
        # zero any slot columns left over from a previous tenant of this slot
        # (handled above: _put_b rewrites the full column block of every target)

    def release(self, adapter: AdapterSet) -> None:
        s = self._owner.pop(id(adapter), None)
        if s is not None:
            self._refs[s] = None

    def layer_ptrs(self, layer: int) -> dict:
        out = {k: v[layer].data_ptr() for k, v in self.t.items()}
        out.update({k: v[layer].data_ptr() for k, v in self.b.items()})
        return out


# ----------------------------------------------------------------------------- runtime
def auto_chunk_pages(max_context: int) -> int:
    """Attention work-item length (pages) for a runtime serving contexts up to max_context:
    16 up to 2.5k tokens (the C2 decode regime), 32 up to 5k, 64 up to 17k, 128 beyond --
    enough (chunk, KV head) items to fill the SMs at long context while each item keeps
    enough 8-page sub-chunks to amortise its start-up, and few enough items that a wide
    shared-prefix batch (C3: 512 query entries per KV head) is not split into many short
    ones. Measured with tools/attn_sweep.py, tools/ablate.py and tools/c3_step_profile.py
    (ICR_CHUNK_PAGES). Fixed per runtime, so a row's attention never depends on which other
    rows share its step."""
    pages = -(-max_context // BLOCK_TOKENS)
    for cp, limit in ((16, 160), (32, 320), (64, 1088)):
        if pages <= limit:
            return cp
    return 128


class Runtime:
    """The device side of one BaseWeights: page arena, adapter slots, block table and the
    C model handle. Sessions borrow a block-table row (sequence slot) each."""

    def __init__(self, base, max_seqs: int = 64, max_context: int = 4096,
                 num_pages: Optional[int] = None, max_rows: int = 512, adapter_slots: int = 8,
                 lora_rank: int = 16, chunk_pages: Optional[int] = None, device="cuda"):
        torch = _torch()
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the B200 path has no CPU fallback")
        cfg = base.config
        cfg.check_device_shapes()
        self.config = cfg
        self.base = base
        self.device = device
        self.max_seqs = max_seqs
        self.max_context = max_context
        self.max_pages_per_seq = (max_context + BLOCK_TOKENS - 1) // BLOCK_TOKENS
        if num_pages is None:
            num_pages = min(max_seqs * self.max_pages_per_seq, 1 << 16)
        self.max_rows = max_rows
        if chunk_pages is None:  # ICR_CHUNK_PAGES: tuning sweeps only (tools/)
            chunk_pages = int(os.environ.get("ICR_CHUNK_PAGES", 0)) or auto_chunk_pages(max_context)
        self.chunk_pages = chunk_pages
        self.dw = base.device(device)
        self.arena = PageArena(cfg, num_pages, device)
        self.slots = AdapterSlots(cfg, adapter_slots, lora_rank if adapter_slots else 0, device)
        self.block_table = np.full((max_seqs, self.max_pages_per_seq), -1, dtype=np.int32)
        self._free_seq = list(range(max_seqs - 1, -1, -1))
        self._handle = C.c_void_p()
        self._lib = _lib.load()
        self._create()

    def check_capacity(self, **caps) -> None:
        for k, v in caps.items():
            have = getattr(self, k, None)
            if have is not None and isinstance(v, int) and v > have:
                raise ConfigError(f"runtime already created with {k}={have} < requested {v}")

    def _create(self) -> None:
        cfg = self.config
        c = _lib.ModelConfigC(
            num_layers=cfg.num_layers, hidden_dim=cfg.hidden_dim, num_heads=cfg.num_heads,
            num_kv_heads=cfg.num_kv_heads, head_dim=cfg.head_dim, ffn_dim=cfg.ffn_dim,
            vocab_size=cfg.vocab_size, rms_eps=cfg.rms_eps, rope_theta=cfg.rope_theta,
            max_positions=self.max_context, num_pages=self.arena.num_pages,
            max_seqs=self.max_seqs, max_pages_per_seq=self.max_pages_per_seq,
            max_rows=self.max_rows, adapter_slots=self.slots.n, lora_rank=self.slots.rank,
            chunk_pages=self.chunk_pages)
        layers = (_lib.LayerWeightsC * cfg.num_layers)()
        for l in range(cfg.num_layers):
            lw = self.dw.layers[l]
            kp, vp = self.arena.layer_ptrs(l)
            ap = self.slots.layer_ptrs(l)
            layers[l] = _lib.LayerWeightsC(
                w_qkv=lw["w_qkv"].data_ptr(), w_o=lw["w_o"].data_ptr(),
                w_gu=lw["w_gu"].data_ptr(), w_down=lw["w_down"].data_ptr(),
                a_q=ap.get("a_q"), b_q=ap.get("b_q"), a_o=ap.get("a_o"), b_o=ap.get("b_o"),
                a_gate=ap.get("a_gate"), a_up=ap.get("a_up"), b_gu=ap.get("b_gu"),
                a_down=ap.get("a_down"), b_down=ap.get("b_down"), k_pages=kp, v_pages=vp)
        self._layers_c = layers
        _lib.check(self._lib.icr_model_create(C.byref(c), layers, self.dw.embed.data_ptr(),
                                              self.dw.lm_head.data_ptr(), C.c_float(1.0),
                                              C.byref(self._handle)))

    def __del__(self):
        try:
            if self._handle:
                self._lib.icr_model_destroy(self._handle)
                self._handle = C.c_void_p()
        except Exception:
            pass

    # -- sequence slots -------------------------------------------------------------------
    def acquire_seq(self) -> int:
        if not self._free_seq:
            raise CapacityError(f"all {self.max_seqs} sequence slots are in use")
        return self._free_seq.pop()

    def release_seq(self, slot: int) -> None:
        self.block_table[slot] = -1
        self._free_seq.append(slot)

    def set_pages(self, slot: int, pages: list) -> None:
        row = self.block_table[slot]
        row[:len(pages)] = pages
        row[len(pages):] = -1

    # -- the step ---------------------------------------------------------------------------
    def forward(self, tokens, kind, seq, pos, adapter, emit, logits: bool = False):
        """One fused forward over token rows (see include/icarus_b200.h icr_batch).
        Returns (tokens for emitting rows, logits tensor or None)."""
        torch = _torch()
        rows = np.array((tokens, kind, seq, pos, adapter, emit), dtype=np.int32)  # one [6, n] block
        n = rows.shape[1]
        n_seqs = int(max(rows[2].max(), 0)) + 1
        base, stride = _lib.addr(rows), rows.strides[0]
        b = _lib.BatchC(n, *[base + i * stride for i in range(6)], _lib.addr(self.block_table), n_seqs)
        n_emit = int(np.count_nonzero(rows[5]))
        out = np.zeros(max(n_emit, 1), dtype=np.int32)
        lg = None
        if logits and n_emit:
            lg = torch.empty(n_emit, self.dw.vocab_pad, dtype=torch.float32, device=self.device)
        _lib.check(self._lib.icr_forward(self._handle, C.byref(b), _lib.addr(out),
                                         lg.data_ptr() if lg is not None else None,
                                         _lib.stream_handle()))
        if lg is not None:
            lg = lg[:, :self.config.vocab_size]
        return out[:n_emit], lg

    def seq_logits(self, slots) -> "torch.Tensor":
        """fp32 logits [n, vocab] of the hidden states the last emitting forwards kept in the
        per-(sequence, kind) store (icr_seq_logits; slot = 2 * seq + kind)."""
        torch = _torch()
        sl = np.ascontiguousarray(slots, dtype=np.int32)
        lg = torch.empty(len(sl), self.dw.vocab_pad, dtype=torch.float32, device=self.device)
        _lib.check(self._lib.icr_seq_logits(self._handle, _lib.i32_ptr(sl), len(sl), lg.data_ptr(),
                                            _lib.stream_handle()))
        return lg[:, :self.config.vocab_size]

    def layer_forward(self, x, layer: int, kind, seq, pos, adapter):
        """One layer of the fused forward (icr_layer_forward) over fp32 rows x [n, d] (device
        tensor); returns the layer's output rows. Encoder rows write this layer's K/V."""
        torch = _torch()
        xin = x.to(self.device, torch.float32).contiguous()
        n = xin.shape[0]
        if xin.ndim != 2 or xin.shape[1] != self.config.hidden_dim:
            from .errors import ShapeError
            raise ShapeError(f"layer input must be [rows, {self.config.hidden_dim}], got {tuple(xin.shape)}")
        rows = np.array((np.zeros(n), kind, seq, pos, adapter, np.zeros(n)), dtype=np.int32)
        n_seqs = int(max(rows[2].max(), 0)) + 1
        base, stride = _lib.addr(rows), rows.strides[0]
        b = _lib.BatchC(n, *[base + i * stride for i in range(6)], _lib.addr(self.block_table), n_seqs)
        out = torch.empty_like(xin)
        _lib.check(self._lib.icr_layer_forward(self._handle, C.byref(b), int(layer), xin.data_ptr(),
                                               out.data_ptr(), _lib.stream_handle()))
        return out

    def decode_loop(self, tokens, kind, seq, pos, adapter, emit, feedback, steps: int):
        """Device-resident decode loop (icr_decode_loop): returns per-step device ms and
        the last step's emitted tokens."""
        arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in (tokens, kind, seq, pos, adapter, emit)]
        n = arrs[0].shape[0]
        n_seqs = int(max(arrs[2].max(), 0)) + 1
        fb = np.ascontiguousarray(feedback, dtype=np.int32)
        b = _lib.BatchC(n, *[_lib.addr(a) for a in arrs], _lib.addr(self.block_table), n_seqs)
        ms = np.zeros(steps, dtype=np.float32)
        last = np.zeros(max(int(np.count_nonzero(arrs[5])), 1), dtype=np.int32)
        _lib.check(self._lib.icr_decode_loop(self._handle, C.byref(b), _lib.i32_ptr(fb), steps,
                                             _lib.i32_ptr(last),
                                             ms.ctypes.data_as(C.POINTER(C.c_float)),
                                             _lib.stream_handle()))
        return ms, last
