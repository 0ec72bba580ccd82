"""Per-CTA timeline of one attention launch (ICR_ATTN_TRACE) at the C4 shape, summarised.

  python tools/attn_trace.py [--ctx 32768] [--adapters 8] [--chunk-pages 128] [--csv out.csv]

Stamps per partial CTA (us from the first stamp): entry, K producer past the PDL wait, Q
loaded, first S ready, softmax loop done, last P.V landed, epilogue done; plus the CTA-0
sub-chunk timeline. Diagnostic only (not a bench number)."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--adapters", type=int, default=8)
    ap.add_argument("--chunk-pages", type=int, default=128)
    ap.add_argument("--csv", default="gpurun_out/attn_trace.csv")
    args = ap.parse_args()
    os.environ["ICR_ATTN_TRACE"] = args.csv
    from tools.attn_sweep import run
    r = run(args.ctx, args.adapters, args.chunk_pages, iters=3)
    print(r)
    rows = [l.strip().split(",") for l in open(args.csv).read().splitlines()[1:]]
    part = np.array([[float(x) for x in l[2:]] for l in rows if l[0] == "partial"])
    merge = np.array([[float(x) for x in l[2:]] for l in rows if l[0] == "merge"])
    sub = [l for l in rows if l[0] == "sub"]
    for l in rows:
        if l[0] == "launch":
            print(f"stamp kernel before the launch {l[2]} us, after it {l[3]} us (relative to the first CTA)")
    names = ["o_final", "q_loaded", "s0_ready", "q_wait", "loop_done", "epi_done", "entry", "k_pdl",
             "published", "cta_end", "merge_go", "merge_done"]
    print(f"partial CTAs {len(part)}")
    for k in (6, 7, 3, 1, 2, 4, 0, 5, 8, 10, 9, 11):
        if k >= part.shape[1]:
            continue
        col = part[:, k]
        col = col[col >= 0]
        if len(col):
            print(f"  {names[k]:10s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
    dur = part[:, 5] - part[:, 6]
    print(f"  CTA duration  min {dur.min():.2f} med {np.median(dur):.2f} max {dur.max():.2f}")
    order = np.argsort(part[:, 6])
    print("  first 4 / last 4 CTAs by entry (entry, end):",
          [(round(part[i, 6], 2), round(part[i, 5], 2)) for i in list(order[:4]) + list(order[-4:])])
    if len(merge):
        w = merge[:, 7][merge[:, 7] >= 0]
        print(f"merge CTAs {len(merge)}: entry min {merge[:, 6].min():.2f}, past the PDL wait "
              f"min {w.min():.2f} med {np.median(w):.2f}, end med {np.median(merge[:, 5]):.2f} "
              f"max {merge[:, 5].max():.2f}")
    if sub:
        print("CTA-0 sub-chunks: j, K issued, S done, P written, PV issued, S->regs, max, pfree, softmax cycles")
        for l in sub[:20]:
            print("  ", l[1:])


if __name__ == "__main__":
    main()
