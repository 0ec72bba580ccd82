"""C4 long-context shared-KV attention sweep (BASELINE.json configs[3]).

Llama-3-8B attention shape (32 query heads, 8 KV heads, hd 128), one layer: N adapted
sequences share one prompt of T tokens (pages shared through the block table) and each
decodes at position T with 2 rows (encoder + decoder). HBM bytes = unique K/V bytes
(T x 8 heads x 128 x 2 x 2 B) -- shared pages counted once -- so GB/s measures whether
pages are really staged once for every model. L2 is flushed between launches.

  python tools/attn_sweep.py [--chunk-pages 16] [--out profiles/attn_sweep.json]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def run(ctx, n_adapters, chunk_pages, iters=5, pipelined=False):
    """pipelined: `iters` launches back to back alternating between two copies of the K/V
    (each larger than L2 at 32K), no flush -- the attention as it runs inside a decode step,
    its page loads overlapping the previous launch's tail. Otherwise L2 is flushed and every
    launch is timed alone."""
    import torch
    from paper_2603_13281_b200 import _lib
    lib = _lib.load()
    H, Hkv, hd = 32, 8, 128
    shared_pages = ctx // 16
    n_pages = shared_pages + n_adapters * 2
    copies = 2 if pipelined else 1
    kp = torch.randn(copies * n_pages, Hkv, 16, hd, device="cuda").to(torch.bfloat16)
    vp = torch.randn(copies * n_pages, Hkv, 16, hd, device="cuda").to(torch.bfloat16)
    mpps = shared_pages + 2
    bt = np.full((n_adapters, mpps), -1, np.int32)
    for s in range(n_adapters):
        bt[s, :shared_pages] = np.arange(shared_pages)
        bt[s, shared_pages] = shared_pages + s  # private tail page holding position ctx
    rows_seq = np.repeat(np.arange(n_adapters, dtype=np.int32), 2)
    rows_pos = np.full(2 * n_adapters, ctx, np.int32)
    q = torch.randn(2 * n_adapters, H * hd, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    flush = None if pipelined else torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    if pipelined:
        iters = max(iters, 20)
    ms = C.c_float()
    span = C.c_float()
    nitems = np.zeros(1, np.int32)
    _lib.check(lib.icr_bench_attention(
        q.data_ptr(), kp.data_ptr(), vp.data_ptr(), H, Hkv, hd, chunk_pages, 2 * n_adapters,
        _lib.i32_ptr(rows_seq), _lib.i32_ptr(rows_pos), _lib.i32_ptr(bt), n_adapters, mpps,
        out.data_ptr(), flush.data_ptr() if flush is not None else None,
        flush.numel() if flush is not None else 0, iters, n_pages if pipelined else 0,
        C.byref(ms), _lib.i32_ptr(nitems), C.byref(span),
        _lib.stream_handle()))
    kv_bytes = (ctx + 1) * Hkv * hd * 2 * 2 + (n_adapters - 1) * Hkv * hd * 2 * 2
    gbs = kv_bytes / (ms.value / 1e3) / 1e9
    del kp, vp, flush
    torch.cuda.empty_cache()
    out = {"context": ctx, "adapters": n_adapters, "ms": ms.value, "unique_kv_bytes": kv_bytes,
           "gbs": gbs, "items": int(nitems[0]), "chunk_pages": chunk_pages,
           "mode": "pipelined" if pipelined else "cold"}
    if not pipelined and span.value > 0:
        out["kernel_span_us"] = span.value
        out["kernel_span_gbs"] = kv_bytes / (span.value / 1e6) / 1e9
    return out


def main():
    from paper_2603_13281_b200.runtime import auto_chunk_pages
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunk-pages", type=int, default=0,
                    help="0: the runtime's rule for the context (runtime.auto_chunk_pages)")
    ap.add_argument("--out", default=None)
    ap.add_argument("--ctx", type=int, default=0, help="single config (profiling)")
    ap.add_argument("--adapters", type=int, default=8)
    ap.add_argument("--pipelined", action="store_true")
    args = ap.parse_args()
    if args.ctx:
        cp = args.chunk_pages or auto_chunk_pages(args.ctx + 16)
        print(json.dumps(run(args.ctx, args.adapters, cp, iters=1, pipelined=args.pipelined)))
        return
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
    res = []
    for ctx in (1024, 2048, 4096, 8192, 16384, 32768):
        for n in (1, 2, 4, 8):
            r = run(ctx, n, args.chunk_pages or auto_chunk_pages(ctx + 16))
            r["frac_of_measured_hbm"] = r["gbs"] / peak
            res.append(r)
            print(json.dumps(r), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps({"peak_hbm_gbs": peak, "results": res}, indent=1))


if __name__ == "__main__":
    main()
