#!/usr/bin/env python
"""Benchmark of the ICaRus multi-model decode hot path on B200 (BASELINE.json configs[1]).

Workload C2: Llama-3-8B-shape random-init base + 8 rank-16 LoRA adapters sharing one
KV cache; one 2048-token prompt prefilled once (adapter 0) and reused by the other seven
through the cross-model prefix pool; then batched fused decode steps (8 encoder rows +
8 decoder rows per step). A "step" = one fused decode step of the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

value      decoder tokens/s, device-resident loop (inputs in HBM, tokens fed back on
           device), CUDA events on the launch stream, max over ranks.
e2e        the same metric through the public API engine.decode_step_batch with host
           tokens: per step H2D of the step's metadata+tokens and D2H of the tokens.
roofline   the gate|up projection GEMM (the dominant tcgen05 kernel, 54% of step bytes)
           re-timed in isolation over all 32 layers; achieved = algorithmic bytes / time.
cpu_baseline  the reference path (oracle port, bitwise equal to the reference) on host
           cores, bounded sample, extrapolated (oracle/cpu_baseline.py).
Multi-GPU: one replica per rank (request batches shard; no collective on the hot path).
"""

from __future__ import annotations

import argparse
import json
import os
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
METRIC = "multi-model decode tokens/s (8 adapters, shared KV)"
WORKLOAD = ("C2: Llama-3-8B-shape random-init + 8 rank-16 LoRA adapters, shared KV, "
            "2k prompt (prefilled once, 7 cross-model prefix hits), batched fused decode")


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


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
            "tok_s": len(per) / t_step, "cores": len(per)}


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
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": res["t_step_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (random weights, uniform token ids)",
        "config": {"workload": WORKLOAD, "model": "llama-3-8b-shape", "adapters": N_ADAPTERS,
                   "rank": RANK, "prompt": PROMPT, "parallelism": "host processes"},
        "cpu_baseline": {"value": res["tok_s"], "unit": "tok/s", "cores": res["cores"],
                         "kind": "port", "sample": sample},
        "e2e": {"value": res["tok_s"], "unit": "tok/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- B200 side
def run_b200(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2603_13281_b200 import _lib
    from paper_2603_13281_b200 import engine as E
    from paper_2603_13281_b200.kvpool import KvCachePool
    from paper_2603_13281_b200.model import AdapterSet, BaseWeights, ModelConfig

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    _lib.load()
    cfg = ModelConfig(**C2)
    K, W = args.steps, args.warmup
    E2E = min(K, 64)
    max_ctx = (PROMPT + W + K + E2E + 32 + 15) // 16 * 16
    base = BaseWeights.on_device(cfg, seed=0)
    adapters = [AdapterSet.on_device(cfg, RANK, ALPHA, seed=1 + i, task=f"agent{i}")
                for i in range(N_ADAPTERS)]
    tail_pages = (max_ctx - PROMPT) // 16 + 2
    rt = base.runtime(max_seqs=N_ADAPTERS + 2, max_context=max_ctx, max_rows=512,
                      adapter_slots=N_ADAPTERS, lora_rank=RANK,
                      num_pages=PROMPT // 16 + N_ADAPTERS * tail_pages + 16)
    pool = KvCachePool(cfg, budget_bytes=4 << 30, mode="icarus")
    prompt = [int(t) for t in np.random.default_rng(1000 + rank).integers(1, cfg.vocab_size, PROMPT)]
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
    hit_tokens = sum(s.ledger.prefix_hit_tokens for s in sessions)

    # ---------------- device-resident loop (value) ----------------
    n = len(sessions)
    for s in sessions:
        s.cache.ensure_pages(PROMPT + W + K - 1)
        rt.set_pages(s.seq, s.cache.pages)
    tok = np.repeat(np.asarray(first, np.int32), 2)
    kind = np.tile(np.asarray([0, 1], np.int32), n)
    seq = np.repeat(np.asarray([s.seq for s in sessions], np.int32), 2)
    adp = np.asarray([x for s in sessions for x in (-1, s.adapter_slot)], np.int32)
    emit = np.ones(2 * n, np.int32)
    fb = np.repeat(np.arange(n, dtype=np.int32) * 2 + 1, 2)
    pos = np.full(2 * n, PROMPT, np.int32)
    _, last = rt.decode_loop(tok, kind, seq, pos, adp, emit, fb, steps=W)
    tok = last[fb]
    pos = pos + W
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        ev0.record(stream)
        step_ms, last = rt.decode_loop(tok, kind, seq, pos, adp, emit, fb, steps=K)
        ev1.record(stream)
        torch.cuda.synchronize()
    elapsed_ms = ev0.elapsed_time(ev1)
    stats = np.zeros(3, np.int64)
    _lib.check(rt._lib.icr_model_stats(rt._handle, stats.ctypes.data_as(
        __import__("ctypes").POINTER(__import__("ctypes").c_int64))))
    launches_per_step = int(stats[0]) + 1  # + the on-device token feedback kernel
    from paper_2603_13281_b200 import dist as D
    elapsed_ms = D.max_over_ranks(elapsed_ms, device="cuda")
    for s in sessions:
        s.cache.advance(W + K)
    value = world * N_ADAPTERS * K / (elapsed_ms / 1e3)
    p95 = D.global_p95([float(x) for x in step_ms])

    # ---------------- end to end through the public API (e2e) ----------------
    toks = [int(t) for t in last[fb[0::2]]]
    torch.cuda.synchronize()
    e2e_lat = []
    t0 = time.perf_counter()
    for _ in range(E2E):
        a = time.perf_counter()
        toks = E.decode_step_batch(sessions, toks)
        e2e_lat.append(time.perf_counter() - a)
    e2e_s = time.perf_counter() - t0
    _lib.check(rt._lib.icr_model_stats(rt._handle, stats.ctypes.data_as(
        __import__("ctypes").POINTER(__import__("ctypes").c_int64))))
    h2d = int(stats[1])
    e2e_value = world * N_ADAPTERS * E2E / D.max_over_ranks(e2e_s, device="cuda")

    # ---------------- roofline of the dominant kernel (gate|up GEMM) ----------------
    import ctypes as C
    kind_ms = (C.c_float * 10)()
    _lib.check(rt._lib.icr_profile_step(rt._handle, kind_ms, _lib.stream_handle()))
    names = ("embed", "qkv", "attention", "o", "gate_up", "down", "lm_gather", "lm_head", "argmax")
    step_breakdown = {n: round(kind_ms[i], 4) for i, n in enumerate(names)}
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
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    traffic = None
    try:
        prof = json.loads((ROOT / "profiles" / "gemm_gu_ncu.json").read_text())
        traffic = prof.get("dram_bytes_per_launch")
    except Exception:
        pass
    # ---------------- C4: long-context shared-KV attention (BASELINE.json configs[3]) ----------
    attn_c4 = None
    if not args.no_attention:
        try:
            from tools.attn_sweep import run as attn_run
            r4 = attn_run(32768, N_ADAPTERS, 128)
            r4p = attn_run(32768, N_ADAPTERS, 128, pipelined=True)
            attn_c4 = {"kernel": "attn_tc_kernel (tcgen05) + attn_merge_kernel",
                       "context": 32768, "adapters": N_ADAPTERS, "chunk_pages": 128,
                       "us": r4["ms"] * 1e3, "unique_kv_bytes": r4["unique_kv_bytes"],
                       "achieved_gbs": r4["gbs"], "frac": r4["gbs"] / float(peaks.get("hbm_gbs", 6650.0)),
                       "l2": "flushed between launches (256 MB read); K/V and q cold, the plan tables re-uploaded after the flush as the engine does every step",
                       "pipelined": {"us": r4p["ms"] * 1e3, "achieved_gbs": r4p["gbs"],
                                     "frac": r4p["gbs"] / float(peaks.get("hbm_gbs", 6650.0)),
                                     "how": "20 launches back to back (PDL), alternating between two copies of the 134 MB K/V (no L2 reuse); per-launch average"}}
        except Exception as exc:  # the C4 line is informative; never fail the bench on it
            attn_c4 = {"error": str(exc)[:200]}
    step_bytes = (rt.dw.nbytes_streamed() + N_ADAPTERS * 73_400_320
                  + (PROMPT + N_ADAPTERS * (W + K // 2)) * cfg.num_layers * 2 * cfg.kv_dim * 2)

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
        "p95_step_ms": p95,
        "prefill_s": prefill_s, "prefix_hit_tokens": hit_tokens,
        "step_hbm_gbs": step_bytes / (elapsed_ms / K / 1e3) / 1e9,
        "clocks": clocks.summary(),
        "e2e": {"value": e2e_value, "unit": "tok/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 4 * 2 * n,
                "p95_step_ms": float(np.sort(e2e_lat)[max(0, int(np.ceil(0.95 * E2E)) - 1)] * 1e3)},
        "gpu_launches": launches_per_step * K,
        "roofline": {"kernel": "gemm_streamk_kernel<16> gate|up (tcgen05, TMA)", "bound": "hbm",
                     "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "avg_launch_ms": avg.value,
                     "algorithmic_bytes_per_launch": gu_bytes,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                     "gemm_launch_us": per_kind},
        "step_breakdown_ms": step_breakdown,
        "attention_c4": attn_c4,
    }
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
    for s in sessions:
        s.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=256)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-attention", action="store_true", help="skip the C4 attention line")
    args = ap.parse_args()
    bad = [k for k in ("ICR_DIAG_NO_LORA", "ICR_SKIP", "ICR_CHUNK_PAGES", "ICR_STAGES", "ICR_PREISSUE",
                       "ICR_LIB_PATH", "ICR_ATTN_MMA") if os.environ.get(k)]
    if bad:  # tuning / diagnostic switches would change (or skip) measured work
        raise SystemExit(f"bench.py refuses to run with {', '.join(bad)} set")
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
