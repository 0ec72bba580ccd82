"""Per-CTA timeline of one CUDA-graph decode step (C2 batch): every GEMM / attention launch
stamps %globaltimer at entry, after the previous kernel completed (griddepcontrol.wait),
and at the end; prints per-launch spans for layer 1 and per-kind medians over all layers.

  python tools/trace_step.py [csv_out]
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import tools.profile_variants as pv  # noqa: E402

KIND = {1: "qkv", 2: "attn", 3: "merge", 4: "o", 5: "gu", 0: "down"}


def analyse(path):
    d = np.genfromtxt(path, delimiter=",", names=True)
    launches = sorted(set(int(x) for x in d["launch"]))
    rows = []
    prev_end = None
    for l in launches:
        x = d[d["launch"] == l]
        entry = x["entry"][x["entry"] >= 0]
        end = x["end"][x["end"] >= 0]
        prev = x["prev_done"][x["prev_done"] >= 0]
        kind = "embed" if l == 0 else (KIND[(l - 1) % 6 + 1 if (l - 1) % 6 + 1 != 6 else 0] if l < 193 else "lm")
        r = dict(l=l, kind=kind, n=len(x), entry0=entry.min(), entry1=entry.max(),
                 prev=np.median(prev) if len(prev) else np.nan, end_med=np.median(end) if len(end) else np.nan,
                 end1=end.max() if len(end) else np.nan)
        r["gap_from_prev_end"] = r["entry0"] - prev_end if prev_end is not None else np.nan
        prev_end = r["end1"]
        rows.append(r)
    for r in rows:
        if 7 <= r["l"] <= 13 or r["l"] >= 190:
            print(f"{r['l']:4d} {r['kind']:6s} ctas {r['n']:4d} entry {r['entry0']:9.2f}..{r['entry1']:9.2f} "
                  f"prev_done {r['prev']:9.2f} end med {r['end_med']:9.2f} max {r['end1']:9.2f}  "
                  f"span {r['end1'] - r['entry0']:7.2f}  gap {r['gap_from_prev_end']:7.2f}")
    print("per kind medians over layers (us): span = last end - first entry; "
          "wait = prev_done - first entry; gap = first entry - previous launch's last end")
    for k in ("qkv", "attn", "merge", "o", "gu", "down"):
        sel = [r for r in rows if r["kind"] == k and r["l"] > 6]
        span = np.median([r["end1"] - r["entry0"] for r in sel])
        wait = np.median([r["prev"] - r["entry0"] for r in sel])
        gap = np.median([r["gap_from_prev_end"] for r in sel])
        body = np.median([r["end1"] - r["prev"] for r in sel])
        print(f"  {k:6s} span {span:7.2f}  wait-for-prev {wait:7.2f}  after-prev-to-end {body:7.2f}  gap {gap:7.2f}")
    # per-SM handoff: when a CTA enters late, what did its SM run before, and when did it exit?
    for l in (10, 11, 12, 13):
        x = d[d["launch"] == l]
        e0 = x["entry"].min()
        late = x[x["entry"] > e0 + 5]
        for c in late[:6]:
            sm = int(c["smid"])
            prev = d[(d["smid"] == sm) & (d["launch"] < l) & (d["launch"] >= l - 3)]
            desc = ", ".join(f"L{int(p['launch'])} end {p['end']:.2f} exit {p['exit']:.2f}" for p in prev)
            print(f"  L{l} cta {int(c['cta'])} sm {sm} entry {c['entry']:.2f}: before on this SM: {desc}")
    total = rows[-1]["end1"] - rows[0]["entry0"]
    print(f"step span {total:.1f} us")


def main():
    from paper_2603_13281_b200 import _lib
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/step_trace.csv"
    if len(sys.argv) > 2 and sys.argv[2] == "--analyse":
        return analyse(out)
    rt = pv.setup()
    _lib.check(rt._lib.icr_profile_trace(rt._handle, out.encode(), _lib.stream_handle()))
    analyse(out)


if __name__ == "__main__":
    main()
