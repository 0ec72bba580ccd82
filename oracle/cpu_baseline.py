"""CPU baseline timing of the reference decode path -- TEST/BENCH INFRASTRUCTURE ONLY.

Times the oracle port (icarus_oracle.py, bitwise equal to the reference) on the host:
the reference is single-threaded numpy whose `_mm` accumulates left to right
(src/tensor.py:151-156), about 3 minutes per Llama-3-8B-shape token. A full step is
therefore infeasible inside a benchmark run; the bounded sample is one fused decode LAYER
at full Llama-3-8B width over a 2048-token context (+ one LM-head product), and a step is
extrapolated as t_step = num_layers * t_layer + t_head.

Only bench.py may import this module.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import icarus_oracle as O


def _layer_session(shape: O.Shape, ctx: int, seed: int) -> O.Session:
    rng = np.random.default_rng(seed)
    d, qd, kvd, f = shape.hidden_dim, shape.q_dim, shape.kv_dim, shape.ffn_dim

    def draw(fan_in, sh):
        return (rng.standard_normal(sh, dtype=np.float32) / np.float32(np.sqrt(fan_in)))

    one = O.Shape(1, d, shape.num_heads, shape.num_kv_heads, shape.head_dim, f, 16,
                  shape.rope_theta, shape.rms_eps)
    w = {"embed": draw(d, (16, d)), "lm_head": draw(d, (d, 16)),
         "final_gain": np.ones(d, np.float32),
         "layers": [{"wq": draw(d, (d, qd)), "wk": draw(d, (d, kvd)), "wv": draw(d, (d, kvd)),
                     "wo": draw(qd, (qd, d)), "gate": draw(d, (d, f)), "up": draw(d, (d, f)),
                     "down": draw(f, (f, d)), "attn_gain": np.ones(d, np.float32),
                     "ffn_gain": np.ones(d, np.float32)}]}
    ad = O.init_adapter(one, seed + 1, rank=16, alpha=32.0)
    for per in ad["layers"]:
        for pair in per.values():
            pair["b"] = (rng.standard_normal(pair["b"].shape, dtype=np.float32) * np.float32(0.05))
    s = O.Session(one, w, ad)
    s.k = [rng.standard_normal((ctx, kvd), dtype=np.float32)]
    s.v = [rng.standard_normal((ctx, kvd), dtype=np.float32)]
    return s


def time_layer_steps(shape: O.Shape, ctx: int, steps: int, warmup: int = 0, seed: int = 0):
    """Per-step seconds of the reference fused decode, one layer at full width."""
    s = _layer_session(shape, ctx, seed)
    tok = 1
    out = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        tok = s.decode_fused(tok % 16)
        dt = time.perf_counter() - t0
        if i >= warmup:
            out.append(dt)
    return out


def time_lm_head(shape: O.Shape, seed: int = 0) -> float:
    """Seconds of the reference LM-head product (1 x d @ d x V through `_mm`)."""
    rng = np.random.default_rng(seed)
    w = rng.standard_normal((shape.hidden_dim, shape.vocab_size), dtype=np.float32)
    x = rng.standard_normal((1, shape.hidden_dim), dtype=np.float32)
    t0 = time.perf_counter()
    O.seq_matmul(x, w)
    return time.perf_counter() - t0


def _worker(args):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    shape, ctx, steps, warmup, seed = args
    return time_layer_steps(shape, ctx, steps, warmup, seed)


def parallel_layer_steps(shape: O.Shape, ctx: int, steps: int, warmup: int, procs: int):
    """One independent oracle session per process (embarrassingly parallel sessions)."""
    import multiprocessing as mp
    ctxm = mp.get_context("spawn")
    with ctxm.Pool(procs) as pool:
        return pool.map(_worker, [(shape, ctx, steps, warmup, 100 + i) for i in range(procs)])
