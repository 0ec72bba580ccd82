"""Model definition: frozen base weights, low-rank adapters, paged KV cache view.

Drop-in for the reference's src/model.py (ModelConfig :36-85, BaseWeights :100-146,
init_base :149-177, LowRankPair/AdapterSet :180-256, KvCacheTensor :259-327).
Same constructor signatures, same seeded draw order, same guards and error classes.

What changes for the B200 path:
  * BaseWeights keeps the reference's frozen float32 host arrays (and freeze hash) and
    adds `device()` -- the packed bf16, K-major, gain-folded layout the kernels stream
    (runtime.py). Llama-3-8B-sized models can be created directly on the device with
    `BaseWeights.on_device` (same distributions; no 32 GB host detour).
  * KvCacheTensor is a block-table view over the shared page arena instead of private
    contiguous arrays: positions live in 16-token pages (BLOCK_TOKENS) that several
    sessions -- several adapted models -- may reference at once. Appends still must come
    from the encoder branch (source_branch 0), exactly as in the reference.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import asdict, dataclass
from typing import Iterator, NamedTuple, Optional

import numpy as np

from .errors import (CapacityError, ConfigError, ContractViolationError, ShapeError,
                     StateError)

DECODER_TARGETS = ("q", "o", "gate", "up", "down")
CONVENTIONAL_TARGETS = ("q", "k", "v", "o", "gate", "up", "down")
BLOCK_TOKENS = 16  # page = pool block (src/kvpool.py:35)

F32 = np.dtype(np.float32)
F64 = np.dtype(np.float64)


@dataclass(frozen=True)
class ModelConfig:
    """Validated shape constants (src/model.py:36-85).

    `precision` keeps the reference's meaning for byte accounting ("f32" default, "f64");
    "bf16" selects 2-byte accounting matching the device KV pages. Device arithmetic is
    always bf16 storage with fp32 accumulation.
    """

    num_layers: int = 4
    hidden_dim: int = 64
    num_heads: int = 4
    num_kv_heads: int = 2
    head_dim: int = 16
    ffn_dim: int = 256
    vocab_size: int = 256
    rope_theta: float = 10000.0
    rms_eps: float = 1e-6
    precision: str = "f32"

    def __post_init__(self):
        for name in ("num_layers", "hidden_dim", "num_heads", "num_kv_heads", "head_dim",
                     "ffn_dim", "vocab_size"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be positive, got {getattr(self, name)}")
        if self.num_heads % self.num_kv_heads != 0:
            raise ConfigError(
                f"num_heads {self.num_heads} not divisible by num_kv_heads {self.num_kv_heads}")
        if self.hidden_dim != self.num_heads * self.head_dim:
            raise ConfigError(f"hidden_dim {self.hidden_dim} != num_heads*head_dim "
                              f"{self.num_heads * self.head_dim}")
        if self.head_dim % 2 != 0:
            raise ConfigError(f"head_dim must be even for rotary embedding, got {self.head_dim}")
        if self.precision not in ("f32", "f64", "bf16"):
            raise ConfigError(f"precision must be f32, f64 or bf16, got {self.precision!r}")
        if self.rms_eps <= 0 or self.rope_theta <= 0:
            raise ConfigError("rms_eps and rope_theta must be positive")

    @property
    def dtype(self) -> np.dtype:
        return F64 if self.precision == "f64" else F32

    @property
    def itemsize(self) -> int:
        return {"f32": 4, "f64": 8, "bf16": 2}[self.precision]

    @property
    def q_dim(self) -> int:
        return self.num_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.num_kv_heads * self.head_dim

    @property
    def kv_bytes_per_token(self) -> int:
        """src/model.py:80-82 (itemsize of the accounting precision)."""
        return self.num_layers * 2 * self.kv_dim * self.itemsize

    @property
    def device_kv_bytes_per_token(self) -> int:
        """Bytes one token occupies in the bf16 page arena."""
        return self.num_layers * 2 * self.kv_dim * 2

    def canonical_json(self) -> str:
        return json.dumps(asdict(self), sort_keys=True)

    def check_device_shapes(self) -> None:
        """The sm_100a kernels tile W rows by 128 and K by 64 (runtime.cu checks again)."""
        qkv = self.q_dim + 2 * self.kv_dim
        if self.head_dim not in (64, 128):
            raise ConfigError(f"B200 attention supports head_dim 64 or 128, got {self.head_dim}")
        if qkv % 128 or self.hidden_dim % 128 or self.ffn_dim % 64:
            raise ConfigError("B200 GEMM tiles need hidden_dim % 128 == 0, ffn_dim % 64 == 0 "
                              "and (q_dim + 2*kv_dim) % 128 == 0")


class Param:
    """Minimal stand-in for the reference's Tensor leaf: `.data`, `.shape`, `.dtype`."""

    __slots__ = ("data", "trainable")

    def __init__(self, data: np.ndarray, trainable: bool = False):
        self.data = data
        self.trainable = trainable

    @property
    def shape(self):
        return self.data.shape

    @property
    def dtype(self):
        return self.data.dtype

    def __repr__(self) -> str:
        return f"Param(shape={self.data.shape}, dtype={self.data.dtype})"


class LayerWeights(NamedTuple):
    wq: Param
    wk: Param
    wv: Param
    wo: Param
    gate: Param
    up: Param
    down: Param
    attn_gain: Param
    ffn_gain: Param


class BaseWeights:
    """Frozen parameter store with a content hash as freeze witness (src/model.py:100-146).

    Host arrays are write-protected at construction; `device()` packs them once into the
    kernel layout. A device-only instance (`on_device`) has no host arrays; its freeze
    witness is a checksum of the device bytes.
    """

    def __init__(self, config: ModelConfig, embed: np.ndarray, layers: list,
                 final_gain: np.ndarray, lm_head: np.ndarray):
        self.config = config

        def freeze(arr) -> Param:
            arr = np.ascontiguousarray(arr, dtype=config.dtype)
            arr.setflags(write=False)
            return Param(arr)

        self.embed = freeze(embed)
        self.layers: list[LayerWeights] = [
            LayerWeights(**{k: freeze(v) for k, v in raw.items()}) for raw in layers]
        self.final_gain = freeze(final_gain)
        self.lm_head = freeze(lm_head)
        self._device = None
        self._runtime = None
        self.seed: Optional[int] = None
        self.freeze_hash = self.content_hash()

    @classmethod
    def on_device(cls, config: ModelConfig, seed: int, device="cuda") -> "BaseWeights":
        """Random-init weights generated directly in the device layout (same N(0,1)/sqrt(fan_in)
        distributions and unit gains as init_base, not byte-equal to numpy's stream)."""
        from .runtime import DeviceWeights
        self = cls.__new__(cls)
        self.config = config
        self.embed = self.lm_head = self.final_gain = None
        self.layers = []
        self._runtime = None
        self.seed = seed
        self._device = DeviceWeights.random(config, seed, device)
        self.freeze_hash = self.content_hash()
        return self

    @property
    def host_resident(self) -> bool:
        return self.embed is not None

    def named(self) -> Iterator[tuple[str, Param]]:
        yield "embed", self.embed
        for i, layer in enumerate(self.layers):
            for name, t in zip(LayerWeights._fields, layer):
                yield f"layers.{i}.{name}", t
        yield "final_gain", self.final_gain
        yield "lm_head", self.lm_head

    def content_hash(self) -> str:
        h = hashlib.sha256()
        h.update(self.config.canonical_json().encode())
        if not self.host_resident:
            h.update(self._device.checksum().encode())
            return h.hexdigest()
        for name, t in self.named():
            h.update(name.encode())
            h.update(str(t.data.shape).encode())
            h.update(t.data.dtype.str.encode())
            h.update(t.data.tobytes())
        return h.hexdigest()

    def verify_frozen(self) -> bool:
        if self.content_hash() != self.freeze_hash:
            return False
        if not self.host_resident:
            return True
        return all(not t.data.flags.writeable for _, t in self.named())

    def device(self, device="cuda"):
        """Packed device copy (bf16, [out, in], gains folded); built once."""
        if self._device is None:
            from .runtime import DeviceWeights
            self._device = DeviceWeights.from_host(self, device)
        return self._device

    def runtime(self, **capacity):
        """The device runtime (page arena, kernel library handle) serving this base."""
        from .runtime import Runtime
        if self._runtime is None:
            self._runtime = Runtime(self, **capacity)
        elif capacity:
            self._runtime.check_capacity(**capacity)
        return self._runtime


def init_base(config: ModelConfig, seed: int) -> BaseWeights:
    """Seeded normal init scaled by 1/sqrt(fan_in), fixed draw order (src/model.py:149-177):
    embed, then per layer wq, wk, wv, wo, gate, up, down, then the LM head."""
    rng = np.random.default_rng(seed)
    dt = config.dtype

    def draw(fan_in: int, shape):
        return (rng.standard_normal(shape) / np.sqrt(fan_in)).astype(dt)

    d, qd, kvd, f = config.hidden_dim, config.q_dim, config.kv_dim, config.ffn_dim
    embed = draw(d, (config.vocab_size, d))
    layers = []
    for _ in range(config.num_layers):
        layers.append({
            "wq": draw(d, (d, qd)), "wk": draw(d, (d, kvd)), "wv": draw(d, (d, kvd)),
            "wo": draw(qd, (qd, d)), "gate": draw(d, (d, f)), "up": draw(d, (d, f)),
            "down": draw(f, (f, d)),
            "attn_gain": np.ones(d, dtype=dt), "ffn_gain": np.ones(d, dtype=dt)})
    lm_head = draw(d, (d, config.vocab_size))
    base = BaseWeights(config, embed, layers, np.ones(d, dtype=dt), lm_head)
    base.seed = seed
    return base


@dataclass
class LowRankPair:
    a: Param  # [rank, in_dim]
    b: Param  # [out_dim, rank]


def _target_dims(config: ModelConfig, target: str) -> tuple[int, int]:
    d, qd, kvd, f = config.hidden_dim, config.q_dim, config.kv_dim, config.ffn_dim
    dims = {"q": (d, qd), "k": (d, kvd), "v": (d, kvd), "o": (qd, d),
            "gate": (d, f), "up": (d, f), "down": (f, d)}
    if target not in dims:
        raise ConfigError(f"unknown adapter target {target!r}; valid: {sorted(dims)}")
    return dims[target]


class AdapterSet:
    """Per-layer low-rank pairs for a fixed set of projection targets (src/model.py:180-256).

    Decoder-side sets cannot name wk/wv/embeddings/norms/LM head: they have no slot. A
    conventional set (with k, v) is accepted here, as in the reference, and refused by
    new_session because it cannot ride a shared cache."""

    def __init__(self, config: ModelConfig, rank: int, alpha: float, targets: tuple,
                 layers: list, task: str = ""):
        if rank < 1:
            raise ConfigError(f"adapter rank must be positive, got {rank}")
        for t in targets:
            _target_dims(config, t)
        if len(layers) != config.num_layers:
            raise ConfigError(
                f"adapter layer count {len(layers)} != model layers {config.num_layers}")
        self.config = config
        self.rank = rank
        self.alpha = alpha
        self.targets = tuple(targets)
        self.layers = layers
        self.task = task
        self.device_seed: Optional[int] = None  # set for device-generated adapters

    @property
    def scaling(self) -> float:
        return self.alpha / self.rank

    @classmethod
    def init(cls, config: ModelConfig, rank: int = 8, alpha: float = 16.0,
             targets: tuple = DECODER_TARGETS, seed: int = 0, task: str = "") -> "AdapterSet":
        """Seeded-normal A, zero B: every adapted projection starts bitwise at its base."""
        rng = np.random.default_rng(seed)
        dt = config.dtype
        layers = []
        for _ in range(config.num_layers):
            per = {}
            for t in targets:
                in_dim, out_dim = _target_dims(config, t)
                a = (rng.standard_normal((rank, in_dim)) / np.sqrt(in_dim)).astype(dt)
                b = np.zeros((out_dim, rank), dtype=dt)
                per[t] = LowRankPair(Param(a, True), Param(b, True))
            layers.append(per)
        return cls(config, rank, alpha, targets, layers, task)

    @classmethod
    def on_device(cls, config: ModelConfig, rank: int, alpha: float, seed: int,
                  b_scale: float = 0.05, task: str = "") -> "AdapterSet":
        """A device-generated adapter with make_agents' distributions (A ~ N/sqrt(in),
        B ~ N(0, b_scale^2)); used for Llama-3-8B-sized benchmarks."""
        self = cls(config, rank, alpha, DECODER_TARGETS, [dict() for _ in range(config.num_layers)],
                   task)
        self.device_seed = seed
        self.b_scale = b_scale
        return self

    def pair(self, layer: int, target: str) -> Optional[LowRankPair]:
        return self.layers[layer].get(target)

    def named_params(self):
        for i, per in enumerate(self.layers):
            for t in sorted(per):
                yield f"layers.{i}.{t}.a", per[t].a
                yield f"layers.{i}.{t}.b", per[t].b

    def params(self) -> list:
        return [p for _, p in self.named_params()]


class KvCacheTensor:
    """Append-only per-layer K/V positions, stored in pages of the shared arena.

    Same contract as the reference (src/model.py:259-327): appends only from the
    encoder branch; written positions are never rewritten; `view` / `rows` / `fingerprint`
    see exactly the written positions. The page table (`pages`) maps position p to
    arena page pages[p // 16], slot p % 16; pages may be shared with other sessions
    (prefix-cache hits) and are reference-counted by the arena.
    """

    def __init__(self, config: ModelConfig, capacity: int, arena=None):
        if capacity < 1:
            raise ConfigError(f"cache capacity must be positive, got {capacity}")
        self.config = config
        self.capacity = capacity
        if arena is None:
            from .runtime import PageArena
            arena = PageArena.host_only(config, pages=(capacity + BLOCK_TOKENS - 1) // BLOCK_TOKENS)
        self.arena = arena
        self.pages: list[int] = []
        self._lengths = [0] * config.num_layers

    def length(self, layer: int = 0) -> int:
        return self._lengths[layer]

    @property
    def position_count(self) -> int:
        return self._lengths[0]

    # -- page management -------------------------------------------------------------
    def ensure_pages(self, upto_position: int) -> None:
        """Map private pages so positions [0, upto_position] are addressable."""
        need = upto_position // BLOCK_TOKENS + 1
        while len(self.pages) < need:
            self.pages.append(self.arena.alloc())

    def attach_shared(self, page_ids: list) -> None:
        """Borrow full pages (a pooled prefix) at the end of an empty-or-page-aligned cache."""
        if self.position_count % BLOCK_TOKENS != 0 or len(self.pages) * BLOCK_TOKENS != self.position_count:
            raise StateError("shared pages attach only at a page boundary")
        for pid in page_ids:
            self.arena.incref(pid)
            self.pages.append(pid)
        n = self.position_count + BLOCK_TOKENS * len(page_ids)
        if n > self.capacity:
            raise CapacityError(f"cache at {self.position_count}/{self.capacity} cannot take "
                                f"{len(page_ids)} more blocks")
        self._lengths = [n] * self.config.num_layers

    def advance(self, n: int) -> None:
        """All layers gained n positions on the device (GPU forward wrote them)."""
        self._lengths = [x + n for x in self._lengths]

    def advance_layer(self, layer: int, n: int) -> None:
        """One layer gained n positions (a single-layer block_forward wrote them)."""
        self._lengths[layer] += n

    def release(self) -> None:
        for pid in self.pages:
            self.arena.decref(pid)
        self.pages = []

    # -- reference API -----------------------------------------------------------------
    def append_block(self, layer: int, k: np.ndarray, v: np.ndarray, source_branch: int) -> None:
        if source_branch != 0:
            raise ContractViolationError(
                f"KV append from branch {source_branch}; only the encoder branch "
                "(0) may produce cache entries")
        expect = (self.config.num_kv_heads, self.config.head_dim)
        if k.ndim != 3 or k.shape[1:] != expect or v.shape != k.shape:
            raise ShapeError(f"append expects [n,{expect[0]},{expect[1]}] pairs, "
                             f"got k {k.shape} v {v.shape}")
        n = k.shape[0]
        at = self._lengths[layer]
        if at + n > self.capacity:
            raise CapacityError(f"cache layer {layer} at {at}/{self.capacity} "
                                f"cannot take {n} more positions")
        if n == 0:
            return
        self.ensure_pages(at + n - 1)
        for p0 in range(at, at + n):
            pid = self.pages[p0 // BLOCK_TOKENS]
            if self.arena.refcount(pid) > 1:
                raise ContractViolationError(f"append into shared page {pid}")
        self.arena.write_rows(layer, self.pages, at, np.asarray(k), np.asarray(v))
        self._lengths[layer] = at + n

    def _gather(self, layer: int, start: int, stop: int):
        return self.arena.read_rows(layer, self.pages, start, stop)

    def view(self, layer: int):
        """Current K/V for one layer as [T, kv_dim] float32 arrays (read from the pages)."""
        t = self._lengths[layer]
        if t == 0:
            raise StateError(f"cache layer {layer} is empty")
        k, v = self._gather(layer, 0, t)
        kv = self.config.kv_dim
        return Param(k.reshape(t, kv)), Param(v.reshape(t, kv))

    def rows(self, layer: int, start: int, stop: int):
        if not (0 <= start < stop <= self._lengths[layer]):
            raise ShapeError(f"rows [{start}:{stop}] outside written range "
                             f"[0:{self._lengths[layer]}]")
        return self._gather(layer, start, stop)

    def fingerprint(self) -> str:
        """sha256 over every written position, all layers, K then V (raw page bytes)."""
        h = hashlib.sha256()
        for layer in range(self.config.num_layers):
            t = self._lengths[layer]
            k, v = self.arena.read_raw(layer, self.pages, 0, t)
            h.update(k)
            h.update(v)
        return h.hexdigest()


# The reference's module-level projection / attention / block functions (src/model.py:334-538),
# computed by the B200 kernels (layers.py).
from .layers import (adapted_linear, base_linear, block_forward, causal_mask,  # noqa: E402,F401
                     decoder_block_readonly, icarus_linear, layer_attention)
