"""TORCH-FP32 ORACLE -- test infrastructure only, never the product path.

A torch float32 restatement of the reference ICaRus decode path (arxiv 2603.13281,
/root/reference/pkg/src/icarus), for shapes the numpy oracle cannot reach in test time
(SURVEY.md §7 H6): Llama-3-8B shape, 32 layers, a 128,256-token vocabulary and a 2k prompt.
Only tests/ may import it.

Same equations as the reference, in the reference's order of operations per layer; the
summation order inside a matmul is torch's (fp32, TF32 disabled), so it is not bitwise equal
to the reference -- it is pinned to the bitwise oracle (oracle/icarus_oracle.py, itself pinned
bytewise to the reference goldens) by tests/test_torch_ref.py (C1, CPU) and by
tests/test_gpu_8b_width.py (one Llama-3-8B-width layer, GPU): max |dlogit| <= 1e-4 * max.

  block_forward prefill   src/model.py:463-478
  block_forward decode    src/model.py:480-506  (K/V from the encoder row, appended before
                                                 attention; icarus_linear on q/o/gate/up/down)
  icarus_linear           src/model.py:355-371  (adapter delta on the decoder row only)
  _lowrank_delta          src/model.py:340-343  scaling * ((x @ A^T) @ B^T)
  layer_attention         src/model.py:384-425  (2H heads; head h uses group (h mod H)//g)
  rope_apply / _rope_trig src/tensor.py:270-318 (interleaved pairs, float64 angles)
  rms_norm                src/tensor.py:217-246
  silu                    src/tensor.py:199-214
  prefill / decode_step_fused / _final_logits  src/engine.py:84-193

Weights are held as [out, in] tensors (any dtype; upcast to fp32 per use) so the B200
runtime's bf16 device weights can be used directly: `from_runtime` untiles them, so the
oracle and the kernels run on IDENTICAL bf16-representable weights.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

NEG_MASK = -1e30  # src/tensor.py:31-33


@dataclass(frozen=True)
class Shape:
    num_layers: int
    hidden_dim: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab_size: int
    rope_theta: float = 10000.0
    rms_eps: float = 1e-6

    @property
    def q_dim(self) -> int:
        return self.num_heads * self.head_dim

    @property
    def kv_dim(self) -> int:
        return self.num_kv_heads * self.head_dim


def _f32(t):
    return t.float() if t.dtype != torch.float32 else t


def linear(x: torch.Tensor, w_out_in: torch.Tensor) -> torch.Tensor:
    """base_linear (src/model.py:334-337): x @ W with W stored transposed ([out, in])."""
    return x @ _f32(w_out_in).T


def rms_norm(x: torch.Tensor, eps: float) -> torch.Tensor:
    """src/tensor.py:217-246 with unit gains (every config's gains are ones; the device
    folds them into the next projection)."""
    inv = 1.0 / torch.sqrt((x * x).mean(dim=1, keepdim=True) + eps)
    return x * inv


def silu(x: torch.Tensor) -> torch.Tensor:
    """src/tensor.py:199-214."""
    return x * torch.sigmoid(x)


class Rope:
    """src/tensor.py:270-318: inv_freq and angles in float64, cast once to float32."""

    def __init__(self, head_dim: int, theta: float, max_pos: int, device):
        half = head_dim // 2
        inv = theta ** (-np.arange(0, half, dtype=np.float64) * 2.0 / head_dim)
        ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
        self.cos = torch.from_numpy(np.cos(ang).astype(np.float32)).to(device)
        self.sin = torch.from_numpy(np.sin(ang).astype(np.float32)).to(device)
        self.hd = head_dim

    def heads(self, x: torch.Tensor, positions: torch.Tensor) -> torch.Tensor:
        """Rotate interleaved (even, odd) pairs of every head of x [n, heads*hd]."""
        n = x.shape[0]
        xv = x.view(n, -1, self.hd)
        ev, od = xv[..., 0::2], xv[..., 1::2]
        c = self.cos[positions][:, None, :]
        s = self.sin[positions][:, None, :]
        out = torch.empty_like(xv)
        out[..., 0::2] = ev * c - od * s
        out[..., 1::2] = ev * s + od * c
        return out.view(n, -1)


@dataclass
class LayerW:
    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    gate: torch.Tensor
    up: torch.Tensor
    down: torch.Tensor


class Weights:
    """Base weights, [out, in] per projection, plus embed [V, d] and lm_head [V, d]."""

    def __init__(self, shape: Shape, embed, layers: list, lm_head):
        self.shape, self.embed, self.layers, self.lm_head = shape, embed, layers, lm_head

    @classmethod
    def from_oracle(cls, shape: Shape, w: dict, device="cpu") -> "Weights":
        """From oracle/icarus_oracle.py's weight dict ([in, out] float32 arrays)."""
        t = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float32).T)).to(device)  # noqa: E731
        layers = [LayerW(*(t(lw[k]) for k in ("wq", "wk", "wv", "wo", "gate", "up", "down")))
                  for lw in w["layers"]]
        return cls(shape, torch.from_numpy(np.array(w["embed"], np.float32)).to(device), layers,
                   t(w["lm_head"]))

    @classmethod
    def from_device(cls, shape: Shape, dw) -> "Weights":
        """From the runtime's packed bf16 DeviceWeights (tile-major, gains folded = ones):
        untiled views of the very bytes the kernels stream."""
        from paper_2603_13281_b200.runtime import untile
        qd, kvd = shape.q_dim, shape.kv_dim
        layers = []
        for lw in dw.layers:
            qkv = untile(lw["w_qkv"])
            gu = untile(lw["w_gu"])
            layers.append(LayerW(qkv[:qd], qkv[qd:qd + kvd], qkv[qd + kvd:], untile(lw["w_o"]),
                                 gu[0::2], gu[1::2], untile(lw["w_down"])))
        return cls(shape, dw.embed, layers, untile(dw.lm_head)[:shape.vocab_size])


class Adapter:
    """Per layer {target: (A [r, in], B [out, r])} and the scaling alpha / r."""

    def __init__(self, layers: list, scaling: float):
        self.layers, self.scaling = layers, scaling

    def pair(self, layer: int, target: str):
        return self.layers[layer].get(target)

    @classmethod
    def from_oracle(cls, ad: dict, device="cpu") -> "Adapter":
        t = lambda a: torch.from_numpy(np.asarray(a, np.float32)).to(device)  # noqa: E731
        return cls([{k: (t(p["a"]), t(p["b"])) for k, p in per.items()} for per in ad["layers"]],
                   float(ad["scaling"]))

    @classmethod
    def from_slots(cls, slots, slot: int) -> "Adapter":
        """From the runtime's resident AdapterSlots: A as uploaded, B already multiplied by
        alpha / r (and rounded to bf16) -- the operands the kernels use -- so scaling = 1."""
        from paper_2603_13281_b200.runtime import untile
        S, r = slots.n, slots.rank
        layers = []
        L = next(iter(slots.t.values())).shape[0]
        for layer in range(L):
            bq, bo = untile(slots.b["b_q"][layer]), untile(slots.b["b_o"][layer])
            bgu, bd = untile(slots.b["b_gu"][layer]), untile(slots.b["b_down"][layer])
            c0, c1 = slot * r, S * r + slot * r
            qd = slots.cfg.q_dim
            layers.append({
                "q": (slots.t["a_q"][layer, slot], bq[:qd, c0:c0 + r]),
                "o": (slots.t["a_o"][layer, slot], bo[:, c0:c0 + r]),
                "gate": (slots.t["a_gate"][layer, slot], bgu[0::2, c0:c0 + r]),
                "up": (slots.t["a_up"][layer, slot], bgu[1::2, c1:c1 + r]),
                "down": (slots.t["a_down"][layer, slot], bd[:, c0:c0 + r])})
        return cls(layers, 1.0)


def lowrank_delta(x, pair, scaling: float):
    """src/model.py:340-343."""
    a, b = pair
    return ((x @ _f32(a).T) @ _f32(b).T) * scaling


class Session:
    """One sequence: per-layer K/V [T, kv_dim] fp32 (src/model.py:259-327) + last logits."""

    def __init__(self, ref: "TorchRef", adapter: Optional[Adapter] = None, capacity: int = 0):
        s = ref.shape
        cap = capacity or ref.max_pos
        self.ref, self.adapter = ref, adapter
        self.k = torch.zeros(s.num_layers, cap, s.kv_dim, device=ref.device)
        self.v = torch.zeros_like(self.k)
        self.length = 0
        self.last_logits: Optional[torch.Tensor] = None

    def copy_prefix(self, other: "Session", n: int) -> None:
        """Pool hit: copy matched K/V rows (src/engine.py:107-111)."""
        self.k[:, :n] = other.k[:, :n]
        self.v[:, :n] = other.v[:, :n]
        self.length = n


class TorchRef:
    def __init__(self, weights: Weights, max_pos: int, device=None):
        self.w = weights
        self.shape = weights.shape
        self.device = device if device is not None else weights.embed.device
        self.max_pos = max_pos
        self.rope = Rope(self.shape.head_dim, self.shape.rope_theta, max_pos, self.device)

    def session(self, adapter: Optional[Adapter] = None, capacity: int = 0) -> Session:
        return Session(self, adapter, capacity)

    # -- attention ----------------------------------------------------------------------
    def attention(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, qpos: torch.Tensor):
        """layer_attention (src/model.py:384-425) for q [n, heads*hd] (heads H or 2H) over
        k, v [T, kv_dim]; scores = (q.k) * f32(1/sqrt(hd)) + mask, softmax, @ v."""
        s = self.shape
        hd, H, grp = s.head_dim, s.num_heads, s.num_heads // s.num_kv_heads
        n, T = q.shape[0], k.shape[0]
        nh = q.shape[1] // hd
        heads = torch.arange(nh, device=q.device)
        g = (heads % H) // grp
        qh = q.view(n, nh, hd).transpose(0, 1)                      # [nh, n, hd]
        kg = k.view(T, s.num_kv_heads, hd).transpose(0, 1)[g]       # [nh, T, hd]
        vg = v.view(T, s.num_kv_heads, hd).transpose(0, 1)[g]
        sc = (qh @ kg.transpose(1, 2)) * np.float32(1.0 / np.sqrt(hd))
        mask = torch.arange(T, device=q.device)[None, :] > qpos[:, None]
        sc = sc + torch.where(mask, torch.tensor(NEG_MASK, device=q.device),
                              torch.tensor(0.0, device=q.device))[None]
        p = torch.softmax(sc, dim=-1)
        return (p @ vg).transpose(0, 1).reshape(n, nh * hd)

    # -- blocks -------------------------------------------------------------------------
    def _append(self, sess: Session, layer: int, k, v, at: int) -> None:
        n = k.shape[0]
        sess.k[layer, at:at + n] = k
        sess.v[layer, at:at + n] = v

    def prefill(self, sess: Session, tokens) -> int:
        """src/engine.py:115-128 over block_forward 'prefill' (src/model.py:463-478)."""
        s, w = self.shape, self.w
        with torch.no_grad():
            toks = torch.as_tensor([int(t) for t in tokens], device=self.device)
            start = sess.length
            pos = torch.arange(start, start + len(toks), device=self.device)
            x = _f32(w.embed[toks]).clone()
            for layer, lw in enumerate(w.layers):
                h = rms_norm(x, s.rms_eps)
                k = self.rope.heads(linear(h, lw.wk), pos)
                v = linear(h, lw.wv)
                self._append(sess, layer, k, v, start)
                q = self.rope.heads(linear(h, lw.wq), pos)
                T = start + len(toks)
                att = self.attention(q, sess.k[layer, :T], sess.v[layer, :T], pos)
                x = x + linear(att, lw.wo)
                h2 = rms_norm(x, s.rms_eps)
                x = x + linear(silu(linear(h2, lw.gate)) * linear(h2, lw.up), lw.down)
            sess.length = start + len(toks)
            final = rms_norm(x[-1:], s.rms_eps)
            sess.last_logits = linear(final, w.lm_head)[0]
            return int(torch.argmax(sess.last_logits))

    def decode_fused(self, sessions: list, tokens: list) -> list:
        """decode_step_fused (src/engine.py:179-193) for several sessions at once: each
        session's pair (encoder row, decoder row) through block_forward 'decode'
        (src/model.py:480-506). The base projections run batched over all pairs (rows are
        independent); LoRA deltas go to decoder rows only, attention is per session."""
        s, w = self.shape, self.w
        n = len(sessions)
        with torch.no_grad():
            toks = torch.as_tensor([int(t) for t in tokens], device=self.device)
            x0 = _f32(w.embed[toks])
            x = torch.stack([x0, x0], 1).reshape(2 * n, s.hidden_dim).clone()  # rows 2i, 2i+1
            pos = torch.as_tensor([ss.length for ss in sessions], device=self.device)
            pos2 = pos.repeat_interleave(2)

            def icarus_linear(xp, wt, layer, target):
                y = linear(xp, wt)
                for i, ss in enumerate(sessions):
                    pair = ss.adapter.pair(layer, target) if ss.adapter is not None else None
                    if pair is not None:
                        y[2 * i + 1] = y[2 * i + 1] + lowrank_delta(xp[2 * i + 1:2 * i + 2], pair,
                                                                    ss.adapter.scaling)[0]
                return y

            for layer, lw in enumerate(w.layers):
                h = rms_norm(x, s.rms_eps)
                h0 = h[0::2]
                k = self.rope.heads(linear(h0, lw.wk), pos)
                v = linear(h0, lw.wv)
                for i, ss in enumerate(sessions):
                    self._append(ss, layer, k[i:i + 1], v[i:i + 1], ss.length)
                q = self.rope.heads(icarus_linear(h, lw.wq, layer, "q"), pos2)
                att = torch.empty(2 * n, s.q_dim, device=self.device)
                for i, ss in enumerate(sessions):
                    T = ss.length + 1
                    q2h = q[2 * i:2 * i + 2].reshape(1, 2 * s.q_dim)
                    a = self.attention(q2h, ss.k[layer, :T], ss.v[layer, :T], pos[i:i + 1])
                    att[2 * i:2 * i + 2] = a.view(2, s.q_dim)
                x = x + icarus_linear(att, lw.wo, layer, "o")
                h2 = rms_norm(x, s.rms_eps)
                f = silu(icarus_linear(h2, lw.gate, layer, "gate")) * icarus_linear(h2, lw.up, layer, "up")
                x = x + icarus_linear(f, lw.down, layer, "down")
            final = rms_norm(x, s.rms_eps)
            logits = linear(final[1::2], w.lm_head)
            out = []
            for i, ss in enumerate(sessions):
                ss.length += 1
                ss.last_logits = logits[i]
                out.append(int(torch.argmax(logits[i])))
            return out


def fp32_matmul():
    """Context: exact fp32 matmuls (no TF32) while the oracle runs."""
    class _Ctx:
        def __enter__(self):
            self.old = (torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32,
                        torch.get_float32_matmul_precision())
            torch.backends.cuda.matmul.allow_tf32 = False
            torch.backends.cudnn.allow_tf32 = False
            torch.set_float32_matmul_precision("highest")
            return self

        def __exit__(self, *exc):
            torch.backends.cuda.matmul.allow_tf32, torch.backends.cudnn.allow_tf32 = self.old[:2]
            torch.set_float32_matmul_precision(self.old[2])
    return _Ctx()
