#!/usr/bin/env python
"""Benchmark of the ICaRus multi-model decode hot path on B200 (BASELINE.json configs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--workload c2|c3|c4|c5] [--no-cpu-baseline] [--no-extras]

--gpus N > 1 without a torchrun environment re-launches itself under
`torch.distributed.run --nproc-per-node N` (one rank per GPU, NCCL); every rank serves its own
replica (requests shard, no collective on the hot path); timings are max over ranks.

Workloads (one JSON line each; the default is the headline, BASELINE.json configs[1]):
  c2  Llama-3-8B-shape random-init base + 8 rank-16 LoRA adapters sharing one KV cache: one
      2048-token prompt prefilled once (adapter 0) and reused by the other seven through the
      cross-model prefix pool, then batched fused decode steps (8 encoder + 8 decoder rows).
      value = decoder tokens/s of the device-resident loop; e2e = the same through
      engine.decode_step_batch with host tokens. At N = 1 the line also carries the C4
      attention kernel (configs[3]), a C4 32k-context decode step, the C3 workflow
      (configs[2]) and the CPU reference port baseline.
  c3  the C3 multi-agent workflow alone (64 requests on a shared 8k prefix, continuous batching).
  c4  the C4 long-context decode step alone (8 adapters on one 32k prompt).
  c5  configs[4]: 512 C3 requests routed over the N ranks (dist.route), each rank serving its
      share; value = all ranks' decoder tokens / slowest rank's wall time, P95 over all requests.
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

C2 = dict(num_layers=32, hidden_dim=4096, num_heads=32, num_kv_heads=8, head_dim=128,
          ffn_dim=14336, vocab_size=128256, rope_theta=5e5, rms_eps=1e-5)
N_ADAPTERS, RANK, ALPHA, PROMPT = 8, 16, 32.0, 2048
C4_CTX = 32768
METRIC = "multi-model decode tokens/s (8 adapters, shared KV)"
WORKLOAD = ("C2: Llama-3-8B-shape random-init + 8 rank-16 LoRA adapters, shared KV, "
            "2k prompt (prefilled once, 7 cross-model prefix hits), batched fused decode")
# algorithmic bytes of one decode step
WEIGHT_BYTES = 15_009_849_344
ADAPTER_BYTES = 73_400_320
KV_BYTES_PER_TOKEN = 131_072


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks() -> dict:
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


def hbm_peak() -> tuple[float, str]:
    p = peaks()
    if "hbm_gbs" in p:
        return float(p["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback 6650 GB/s (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][1]) if self.rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- CPU side
def cpu_baseline_sample(procs: int, steps: int, warmup: int):
    """Reference fused decode (oracle port) at Llama-3-8B width: bounded sample."""
    from oracle import cpu_baseline as B
    from oracle import icarus_oracle as O
    sh = O.Shape(**{k: C2[k] for k in ("num_layers", "hidden_dim", "num_heads", "num_kv_heads",
                                       "head_dim", "ffn_dim", "vocab_size", "rope_theta",
                                       "rms_eps")})
    if procs <= 1:
        per = [B.time_layer_steps(sh, PROMPT, steps, warmup)]
    else:
        per = B.parallel_layer_steps(sh, PROMPT, steps, warmup, procs)
    t_head = B.time_lm_head(sh)
    t_layer = statistics.median([t for run in per for t in run])
    t_step = C2["num_layers"] * t_layer + t_head
    return {"t_layer_s": t_layer, "t_head_s": t_head, "t_step_s": t_step,
            "tok_s": len(per) / t_step, "cores": len(per), "layer_steps": steps * len(per)}


def c1_direct() -> dict:
    """BASELINE.json configs[0] (C1) on the reference port, timed directly (no extrapolation):
    one prefill of 128 tokens, then 32 fused decode steps of one adapter, 1 core."""
    from oracle import icarus_oracle as O
    shape = O.Shape(num_layers=2, hidden_dim=256, num_heads=2, num_kv_heads=1, head_dim=128,
                    ffn_dim=1024, vocab_size=1024)
    w = O.init_base(shape, 0)
    ad = O.make_agents(shape, 2, seed=1)[0]
    s = O.Session(shape, w, ad)
    prompt = [int(t) for t in np.random.default_rng(0).integers(1, 1024, 128)]
    t0 = time.perf_counter()
    tok = s.prefill(prompt)
    pre = time.perf_counter() - t0
    lat = []
    for _ in range(32):
        a = time.perf_counter()
        tok = s.decode_fused(tok)
        lat.append(time.perf_counter() - a)
    from paper_2603_13281_b200.dist import p95_nearest_rank
    return {"config": "C1 (configs[0]): 2 layers, d 256, 128-token prompt, 32 fused decode steps",
            "decode_tok_s": len(lat) / sum(lat), "p95_step_ms": p95_nearest_rank(lat) * 1e3,
            "prefill_s": pre, "cores": 1, "extrapolated": False}


def host_procs() -> int:
    n = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available / 2 ** 30
        n = min(n, max(1, int((avail - 8) // 2.5)))
    except Exception:
        pass
    return max(1, min(n, 64))


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    procs = host_procs()
    # one reference layer-step is ~6 s of CPU: bound the sample so the run ends in minutes
    steps, warm = min(args.steps, 6), min(args.warmup, 1)
    res = cpu_baseline_sample(procs, steps, warm)
    sample = (f"{res['cores']} independent oracle sessions (one per core), each a fused decode "
              f"of 1 of 32 layers at Llama-3-8B width over a 2048-token context, "
              f"{steps} timed layer-steps after {warm} warm-up; + LM head once; "
              f"t_step = 32*t_layer + t_head = {res['t_step_s']:.2f} s (extrapolated)")
    line = {
        "impl": "reference", "metric": METRIC, "value": res["tok_s"], "unit": "tok/s",
        "n_gpus": world, "steps": steps, "steps_requested": args.steps, "warmup": warm,
        "extrapolated": True,
        "ms_per_step": res["t_step_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (random weights, uniform token ids)",
        "config": {"workload": WORKLOAD, "model": "llama-3-8b-shape", "adapters": N_ADAPTERS,
                   "lora_rank": RANK, "prompt": PROMPT, "rows_per_step": 2 * N_ADAPTERS,
                   "parallelism": "host processes (one reference session per core)"},
        "cpu_baseline": {"value": res["tok_s"], "unit": "tok/s", "cores": res["cores"],
                         "kind": "port", "sample": sample},
        "e2e": {"value": res["tok_s"], "unit": "tok/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "c1_direct": c1_direct(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 side
def _stats(rt):
    import ctypes as C
    from paper_2603_13281_b200 import _lib
    st = np.zeros(3, np.int64)
    _lib.check(rt._lib.icr_model_stats(rt._handle, st.ctypes.data_as(C.POINTER(C.c_int64))))
    return st


def build_models(device_seed: int = 0):
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig
    cfg = ModelConfig(**C2)
    base = BaseWeights.on_device(cfg, seed=device_seed)
    adapters = [AdapterSet.on_device(cfg, RANK, ALPHA, seed=1 + i, task=f"agent{i}")
                for i in range(N_ADAPTERS)]
    return cfg, base, adapters


def shared_prompt_sessions(cfg, base, adapters, rt, prompt, max_ctx):
    """Prefill the prompt once (adapter 0), commit it to an icarus pool, prefill the other
    adapters through the pool (full cross-model prefix hits). Returns (sessions, first tokens,
    prefill seconds, hit tokens)."""
    import torch

    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.kvpool import KvCachePool
    pool = KvCachePool(cfg, budget_bytes=64 << 30, mode="icarus")
    sessions = [E.new_session(base, a, max_ctx, runtime=rt) for a in adapters]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    first = [E.prefill(sessions[0], prompt, pool=pool, reader="agent0")]
    torch.cuda.synchronize()
    prefill_s = time.perf_counter() - t0
    pool.commit(None, prompt, sessions[0].cache,
                next_token_fn=lambda p: E.base_next_token_at(sessions[0], p), creator="agent0")
    for i, s in enumerate(sessions[1:], 1):
        first.append(E.prefill(s, prompt, pool=pool, reader=f"agent{i}"))
    hit = sum(s.ledger.prefix_hit_tokens for s in sessions)
    return sessions, first, prefill_s, hit, pool


def device_loop(rt, sessions, first, start_pos, steps):
    """icr_decode_loop over the sessions' fused pairs: per-step device ms, last tokens."""
    n = len(sessions)
    tok = np.repeat(np.asarray(first, np.int32), 2)
    kind = np.tile(np.asarray([0, 1], np.int32), n)
    seq = np.repeat(np.asarray([s.seq for s in sessions], np.int32), 2)
    adp = np.asarray([x for s in sessions for x in (-1, s.adapter_slot)], np.int32)
    emit = np.ones(2 * n, np.int32)
    fb = np.repeat(np.arange(n, dtype=np.int32) * 2 + 1, 2)
    pos = np.full(2 * n, start_pos, np.int32)
    ms, last = rt.decode_loop(tok, kind, seq, pos, adp, emit, fb, steps=steps)
    return ms, last[fb[0::2]]


def attention_c4(peak: float) -> dict:
    """C4 (configs[3]) shared-KV attention alone at 32k context x 8 adapters (one layer's
    launch: tcgen05 partial kernel + merge)."""
    from tools.attn_sweep import run as attn_run
    r = attn_run(C4_CTX, N_ADAPTERS, 128)
    rp = attn_run(C4_CTX, N_ADAPTERS, 128, pipelined=True)
    kv = r["unique_kv_bytes"]
    span_us = r.get("kernel_span_us")
    out = {
        "kernel": "attn_tc_kernel (persistent tcgen05, TMA) + attn_merge_kernel",
        "context": C4_CTX, "adapters": N_ADAPTERS, "chunk_pages": 128,
        "unique_kv_bytes": kv, "peak_gbs": peak,
        "device_span": {"us": span_us, "achieved_gbs": kv / (span_us / 1e6) / 1e9 if span_us else None,
                        "frac": (kv / (span_us / 1e6) / 1e9 / peak) if span_us else None,
                        "how": "L2 flushed (256 MB read) before each launch, plan tables re-uploaded; "
                               "%globaltimer from the first partial CTA's start to the last partial/merge "
                               "CTA's end (the kernels' own duration, no event or launch overhead)"},
        "pipelined": {"us": rp["ms"] * 1e3, "achieved_gbs": rp["gbs"], "frac": rp["gbs"] / peak,
                      "how": "20 launches back to back (PDL), alternating between two copies of the "
                             "134 MB K/V (no L2 reuse) -- how the attention runs inside a decode step; "
                             "CUDA events, per-launch average"},
        "cold_events": {"us": r["ms"] * 1e3, "achieved_gbs": r["gbs"], "frac": r["gbs"] / peak,
                        "how": "CUDA events around one cold launch (includes launch latency)"},
    }
    out["frac"] = out["device_span"]["frac"]
    return out


def prefill_warm(cfg, base, adapters) -> dict:
    """warm prefill of 2k and 8k-token prompts through the public API
    (engine.prefill, an adapted session, no pool hit, every token computed), 512-row forwards
    of the decode kernels (bitwise equal to decode). Median of 3 after one untimed call (the
    bench line's prefill_s is the very first, cold call: graph capture included). Tensor-bound:
    FLOPs = 2 * tokens * (linear params) + causal attention (4 * hd * heads * T^2 / 2 per layer)."""
    import torch

    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.runtime import Runtime
    p = peaks()
    peak_tf = float(p.get("bf16_tflops_sustained", 0) or 0) or 1385.2
    out = {"how": "engine.prefill of a fresh adapted session (no pool), median of 3 warm calls",
           "peak_tflops": peak_tf, "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained"}
    rt = Runtime(base, max_seqs=2, max_context=8192 + 64, max_rows=512, adapter_slots=N_ADAPTERS,
                 lora_rank=RANK, num_pages=2 * (8192 // 16) + 16)
    d, qd, kvd = cfg.hidden_dim, cfg.num_heads * cfg.head_dim, cfg.num_kv_heads * cfg.head_dim
    lin = cfg.num_layers * ((qd + 2 * kvd) * d + d * qd + 3 * cfg.ffn_dim * d)  # linear params
    for T in (2048, 8192):
        prompt = [int(t) for t in np.random.default_rng(T).integers(1, cfg.vocab_size, T)]
        times = []
        for it in range(4):
            s = E.new_session(base, adapters[0], T + 16, runtime=rt)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            E.prefill(s, prompt)
            torch.cuda.synchronize()
            if it:
                times.append(time.perf_counter() - t0)
            s.close()
        sec = float(np.median(times))
        flops = 2.0 * T * lin + cfg.num_layers * 4.0 * cfg.head_dim * cfg.num_heads * T * T / 2
        out[f"{T}"] = {"s": sec, "tok_s": T / sec, "tflops": flops / sec / 1e12,
                       "frac_of_tensor_peak": flops / sec / 1e12 / peak_tf}
    del rt
    torch.cuda.empty_cache()
    return out


def c4_decode(cfg, base, adapters, steps: int, warmup: int, peak: float) -> dict:
    """C4 (configs[3]) as a decode step: 8 adapters on one 32k-token prompt (prefilled once,
    7 cross-model prefix hits), full 32-layer fused decode steps."""
    import ctypes as C

    import torch

    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200.runtime import Runtime
    max_ctx = C4_CTX + warmup + steps + 32
    tail = (max_ctx - C4_CTX) // 16 + 2
    rt = Runtime(base, max_seqs=N_ADAPTERS + 2, max_context=max_ctx, max_rows=512,
                 adapter_slots=N_ADAPTERS, lora_rank=RANK,
                 num_pages=C4_CTX // 16 + N_ADAPTERS * tail + 16)
    prompt = [int(t) for t in np.random.default_rng(4000).integers(1, cfg.vocab_size, C4_CTX)]
    sessions, first, prefill_s, hit, _ = shared_prompt_sessions(cfg, base, adapters, rt, prompt, max_ctx)
    for s in sessions:
        s.cache.ensure_pages(C4_CTX + warmup + steps - 1)
        rt.set_pages(s.seq, s.cache.pages)
    _, toks = device_loop(rt, sessions, first, C4_CTX, warmup)
    torch.cuda.synchronize()
    ms, _ = device_loop(rt, sessions, toks, C4_CTX + warmup, steps)
    step_ms = float(np.sum(ms)) / steps
    kind_ms = (C.c_float * 10)()
    _lib.check(rt._lib.icr_profile_step(rt._handle, kind_ms, _lib.stream_handle()))
    step_bytes = (WEIGHT_BYTES + N_ADAPTERS * ADAPTER_BYTES
                  + (C4_CTX + N_ADAPTERS * (warmup + steps // 2)) * KV_BYTES_PER_TOKEN)
    for s in sessions:
        s.close()
    out = {"workload": "C4 (configs[3]): 8 rank-16 adapters on one 32k-token prompt, fused decode",
           "decode_tok_s": N_ADAPTERS / (step_ms / 1e3), "ms_per_step": step_ms,
           "steps": steps, "prefill_32k_s": prefill_s, "prefix_hit_tokens": hit,
           "step_bytes": step_bytes, "achieved_gbs": step_bytes / (step_ms / 1e3) / 1e9,
           "frac_of_hbm_roofline": step_bytes / (step_ms / 1e3) / 1e9 / peak,
           "roofline_tok_s": N_ADAPTERS / (step_bytes / (peak * 1e9)),
           "serial_profile_ms": {"attention_32_launches": round(kind_ms[2], 4),
                                 "per_attention_launch_us": round(kind_ms[2] / 32 * 1e3, 2),
                                 "total_serial": round(kind_ms[9], 4)}}
    del rt
    torch.cuda.empty_cache()
    return out


def run_workflow(cfg, base, adapters, requests: int, world: int, rank: int, peak: float) -> dict:
    """C3 / C5 serving over the fused step (paper_2603_13281_b200.workflow): requests routed
    over the ranks by prefix affinity (dist.route), each rank serving its share."""
    import torch

    from paper_2603_13281_b200 import dist as D
    from paper_2603_13281_b200 import workflow as W
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.runtime import Runtime
    wcfg = W.WorkflowConfig(requests=requests, prefix_len=8192, max_batch=64)
    prefix, reqs = W.make_workload(wcfg, cfg.vocab_size)
    mine = D.shard(reqs, world, rank, prompts=[list(prefix) + list(r.turns[0].new_tokens) for r in reqs])
    need = W.max_context_tokens(prefix, reqs)
    max_ctx = (need + 64 + 15) // 16 * 16
    live = min(len(mine), wcfg.max_batch)
    private_pages = (need - wcfg.prefix_len) // 16 + 8
    num_pages = wcfg.prefix_len // 16 + live * private_pages * 2 + 64
    rt = Runtime(base, max_seqs=live * 2 + 8, max_context=max_ctx, max_rows=512,
                 adapter_slots=N_ADAPTERS, lora_rank=RANK, num_pages=num_pages)
    # the pool's budget is in the reference's accounting units (kv_bytes_per_token of the
    # config precision, src/kvpool.py:78-120): one block per arena page
    pool = KvCachePool(cfg, budget_bytes=num_pages * cfg.kv_bytes_per_token * 16, mode="icarus")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    W.warm_prefix(base, pool, prefix, max_ctx, runtime=rt)
    torch.cuda.synchronize()
    prefix_s = time.perf_counter() - t0
    rep = W.serve(base, adapters, pool, prefix, mine, wcfg, max_ctx, runtime=rt)
    wall = D.max_over_ranks(rep.wall_s, device="cuda")
    tokens = D.sum_over_ranks(rep.decoder_tokens, device="cuda")
    steps = D.sum_over_ranks(rep.decode_steps, device="cuda")
    p95 = D.global_p95(rep.latencies_ms)
    # roofline: per fused step the weights + adapters stream once, the shared
    # prefix KV once and every live sequence's private KV once
    avg_live = rep.decoder_tokens / max(rep.decode_steps, 1)
    avg_private = 0.5 * (need - wcfg.prefix_len)
    step_bytes = (WEIGHT_BYTES + N_ADAPTERS * ADAPTER_BYTES + wcfg.prefix_len * KV_BYTES_PER_TOKEN
                  + avg_live * avg_private * KV_BYTES_PER_TOKEN)
    bound_tok_s = avg_live / (step_bytes / (peak * 1e9))
    out = {"requests": requests, "ranks": world, "requests_this_rank": len(mine),
           "decode_tok_s": tokens / wall, "p95_request_latency_ms": p95, "wall_s": wall,
           "prefix_prefill_s": prefix_s, "decode_steps": int(steps), "decoder_tokens": int(tokens),
           "avg_live_sequences": avg_live, "prefix_hit_tokens": rep.prefix_hit_tokens,
           "cross_model_hit_tokens": rep.cross_model_hit_tokens, "turns": rep.turns,
           "roofline": {"step_bytes_model": step_bytes, "bound_tok_s_per_rank": bound_tok_s,
                        "frac": (tokens / wall / world) / bound_tok_s,
                        "note": "HBM-bound per rank: weights + adapters + shared prefix KV once per "
                                "step + each live sequence's private KV (BASELINE.md section 4)"}}
    del rt
    torch.cuda.empty_cache()
    return out


def run_b200(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200 import dist as D
    from paper_2603_13281_b200 import engine as E

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.load()
    peak, peak_src = hbm_peak()
    cfg, base, adapters = build_models()
    K, W = args.steps, args.warmup

    if args.workload in ("c3", "c5"):
        requests = 64 if args.workload == "c3" else 512
        with ClockSampler(local) as clocks:
            res = run_workflow(cfg, base, adapters, requests, world, rank, peak)
        if rank == 0:
            print(json.dumps({
                "metric": "multi-agent workflow decode tokens/s (8 adapters, shared 8k prefix)",
                "value": res["decode_tok_s"], "unit": "tok/s", "n_gpus": world, "steps": res["decode_steps"],
                "warmup": 0, "ms_per_step": res["wall_s"] * 1e3 / max(res["decode_steps"] / world, 1),
                "higher_is_better": True, "scaling": "strong" if args.workload == "c5" else "weak",
                "vs_baseline": None, "dtype": "bf16",
                "data": "synthetic (random-init Llama-3-8B-shape weights and adapters, generated workload)",
                "config": {"workload": f"{args.workload.upper()}: {requests} requests, shared 8k prefix, "
                                       "8 rank-16 adapters round-robin over 2-4 turns",
                           "parallelism": f"dp{world} (requests routed by prefix affinity, no collective)"},
                "p95_request_latency_ms": res["p95_request_latency_ms"], "detail": res,
                "e2e": {"value": res["decode_tok_s"], "unit": "tok/s",
                        "note": "serve() drives the public engine API with host tokens: the whole "
                                "run is end to end"},
                "clocks": clocks.summary()}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    if args.workload == "c4":
        with ClockSampler(local) as clocks:
            res = c4_decode(cfg, base, adapters, K, W, peak)
        tok_s = D.sum_over_ranks(res["decode_tok_s"], device="cuda") if world > 1 else res["decode_tok_s"]
        if rank == 0:
            print(json.dumps({"metric": METRIC + " at 32k context", "value": tok_s, "unit": "tok/s",
                              "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": res["ms_per_step"],
                              "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                              "dtype": "bf16", "data": "synthetic", "config": {"workload": res["workload"]},
                              "detail": res, "clocks": clocks.summary()}), flush=True)
        if world > 1:
            dist.destroy_process_group()
        return

    # ---------------- C2: the headline ----------------
    E2E = min(K, 64)
    max_ctx = (PROMPT + W + K + W + E2E + 32 + 15) // 16 * 16
    tail_pages = (max_ctx - PROMPT) // 16 + 2
    rt = base.runtime(max_seqs=N_ADAPTERS + 2, max_context=max_ctx, max_rows=512,
                      adapter_slots=N_ADAPTERS, lora_rank=RANK,
                      num_pages=PROMPT // 16 + N_ADAPTERS * tail_pages + 16)
    prompt = [int(t) for t in np.random.default_rng(1000 + rank).integers(1, cfg.vocab_size, PROMPT)]
    sessions, first, prefill_s, hit_tokens, _ = shared_prompt_sessions(cfg, base, adapters, rt,
                                                                       prompt, max_ctx)
    n = len(sessions)
    for s in sessions:
        s.cache.ensure_pages(PROMPT + W + K - 1)
        rt.set_pages(s.seq, s.cache.pages)
    _, toks = device_loop(rt, sessions, first, PROMPT, W)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        step_ms, toks = device_loop(rt, sessions, toks, PROMPT + W, K)
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = D.max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    launches_per_step = int(_stats(rt)[0]) + 1  # + the on-device token feedback kernel
    for s in sessions:
        s.cache.advance(W + K)
    value = world * N_ADAPTERS * K / (elapsed_ms / 1e3)
    p95 = D.global_p95([float(x) for x in step_ms])

    # ---------------- end to end through the public API (e2e) ----------------
    toks = [int(t) for t in toks]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(W):  # untimed: the public-API path's first calls (graph capture for the
        toks = E.decode_step_batch(sessions, toks)  # step shapes the device loop did not use)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e2e_lat = []
    t0 = time.perf_counter()
    for _ in range(E2E):
        a = time.perf_counter()
        toks = E.decode_step_batch(sessions, toks)
        e2e_lat.append(time.perf_counter() - a)
    e2e_s = D.max_over_ranks(time.perf_counter() - t0, device="cuda")
    h2d = int(_stats(rt)[1])
    e2e_value = world * N_ADAPTERS * E2E / e2e_s

    # ---------------- roofline of the dominant kernel (gate|up GEMM) ----------------
    import ctypes as C
    kind_ms = (C.c_float * 10)()
    _lib.check(rt._lib.icr_profile_step(rt._handle, kind_ms, _lib.stream_handle()))
    names = ("embed", "qkv", "attention", "o", "gate_up", "down", "lm_gather", "lm_head", "argmax")
    step_breakdown = {nm: round(kind_ms[i], 4) for i, nm in enumerate(names)}
    step_breakdown["total_serial"] = round(kind_ms[9], 4)
    avg = C.c_float()
    per_kind = {}
    for which, name in ((0, "o"), (2, "down"), (3, "lm_head"), (1, "gate_up")):
        _lib.check(rt._lib.icr_profile_gemm(rt._handle, which, 2, C.byref(avg), _lib.stream_handle()))
        per_kind[name] = round(avg.value * 1e3, 2)
    rows = 2 * n
    gu_bytes = (2 * cfg.ffn_dim * cfg.hidden_dim * 2 + rows * cfg.hidden_dim * 2
                + rows * cfg.ffn_dim * 2 + N_ADAPTERS * 2 * cfg.ffn_dim * RANK * 2)
    achieved = gu_bytes / (avg.value / 1e3) / 1e9
    traffic = None
    try:
        traffic = json.loads((ROOT / "profiles" / "gemm_gu_ncu.json").read_text()).get("dram_bytes_per_launch")
    except Exception:
        pass
    step_bytes = (WEIGHT_BYTES + N_ADAPTERS * ADAPTER_BYTES
                  + (PROMPT + N_ADAPTERS * (W + K // 2)) * KV_BYTES_PER_TOKEN)
    for s in sessions:
        s.close()

    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init Llama-3-8B-shape weights and adapters, uniform token ids)",
        "config": {"workload": WORKLOAD, "model": "llama-3-8b-shape", "adapters": N_ADAPTERS,
                   "lora_rank": RANK, "prompt": PROMPT, "rows_per_step": 2 * n,
                   "context": [PROMPT + W, PROMPT + W + K],
                   "l2": "no flush needed: each step streams 15.6 GB of weights >> 126 MB L2",
                   "parallelism": f"dp{world} (independent replicas, no collective)"},
        "ranks": {"world_size": world, "backend": "nccl" if world > 1 else None,
                  "nccl_world_size": dist.get_world_size() if world > 1 else None},
        "p95_step_ms": p95,
        "prefill_s": prefill_s, "prefill_tok_s": PROMPT / prefill_s, "prefix_hit_tokens": hit_tokens,
        "step_hbm_gbs": step_bytes / (elapsed_ms / K / 1e3) / 1e9,
        "step_roofline_frac": step_bytes / (elapsed_ms / K / 1e3) / 1e9 / peak,
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4 * 2 * n,
                "p95_step_ms": float(np.sort(e2e_lat)[max(0, int(np.ceil(0.95 * E2E)) - 1)] * 1e3)},
        "gpu_launches": launches_per_step * K,
        "roofline": {"kernel": "gemm_streamk_kernel<16> gate|up (tcgen05, TMA)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "avg_launch_ms": avg.value,
                     "algorithmic_bytes_per_launch": gu_bytes, "peak_source": peak_src,
                     "traffic_source": "profiles/gemm_gu_ncu.json (ncu --set full of this kernel)",
                     "gemm_launch_us": per_kind},
        "step_breakdown_ms": step_breakdown,
    }
    if world == 1 and not args.no_extras:
        for key, fn in (("prefill_warm", lambda: prefill_warm(cfg, base, adapters)),
                        ("attention_c4", lambda: attention_c4(peak)),
                        ("c4_decode", lambda: c4_decode(cfg, base, adapters, 32, 3, peak)),
                        ("c3", lambda: run_workflow(cfg, base, adapters, 64, 1, 0, peak))):
            try:
                line[key] = fn()
            except Exception as exc:  # the extra lines are informative; never fail the bench
                line[key] = {"error": f"{type(exc).__name__}: {str(exc)[:300]}"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = cpu_baseline_sample(1, 2, 0)
        line["cpu_baseline"] = {
            "value": res["tok_s"], "unit": "tok/s", "cores": 1, "kind": "port",
            "sample": (f"oracle port (bitwise = reference) on 1 core: 2 fused decode steps of 1 of "
                       f"32 layers at Llama-3-8B width, 2048 ctx ({res['t_layer_s']:.2f} s/layer) + "
                       f"LM head ({res['t_head_s']:.2f} s); t_step extrapolated "
                       f"{res['t_step_s']:.1f} s for one session")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2", choices=["c2", "c3", "c4", "c5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the C4 attention / C4 step / C3 sub-lines of the C2 run")
    args = ap.parse_args()
    bad = [k for k in ("ICR_DIAG_NO_LORA", "ICR_SKIP", "ICR_CHUNK_PAGES", "ICR_STAGES", "ICR_PREISSUE",
                       "ICR_LIB_PATH", "ICR_ATTN_MMA") if os.environ.get(k)]
    if bad:  # tuning / diagnostic switches would change (or skip) measured work
        raise SystemExit(f"bench.py refuses to run with {', '.join(bad)} set")
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.gpus > 1 and world == 0:
        # one rank per GPU: re-launch under torch.distributed.run on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(free_port()), str(Path(__file__).resolve())] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if world and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} disagrees with WORLD_SIZE {world}")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
