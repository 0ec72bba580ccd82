"""Per-kind phase medians of a trace CSV written by icr_profile_trace (tools/trace_step.py):
for every GEMM launch, times relative to the launch's prev_done median (griddepcontrol.wait
return): entry spread, producer issued_all, last MMA commit, epilogue done, CTA end, CTA exit.

  python tools/trace_phases.py gpurun_out/trace.csv
"""
import sys

import numpy as np

KIND = {1: "qkv", 2: "attn", 3: "merge", 4: "o", 5: "gu", 0: "down"}


def main(path):
    d = np.genfromtxt(path, delimiter=",", names=True)
    launches = sorted(set(int(x) for x in d["launch"]))
    acc = {}
    for l in launches:
        if l == 0 or l >= 193:
            continue
        k = (l - 1) % 6 + 1
        kind = KIND[k if k != 6 else 0]
        x = d[d["launch"] == l]
        pd = np.median(x["prev_done"][x["prev_done"] >= 0]) if (x["prev_done"] >= 0).any() else np.nan

        def rel(col, f=np.median):
            v = x[col][x[col] >= 0]
            return f(v) - pd if len(v) else np.nan
        row = dict(entry_min=rel("entry", np.min), entry_max=rel("entry", np.max),
                   issued_med=rel("issued_all"), issued_max=rel("issued_all", np.max),
                   mma_max=rel("mma_last_commit", np.max), epi_done_max=rel("epi_done", np.max),
                   end_med=rel("end"), end_max=rel("end", np.max), exit_med=rel("exit"),
                   exit_max=rel("exit", np.max),
                   exit_minus_end_med=np.median(x["exit"] - x["end"]),
                   exit_minus_end_max=np.max(x["exit"] - x["end"]))
        acc.setdefault(kind, []).append(row)
    keys = list(next(iter(acc.values()))[0].keys())
    print("kind   " + " ".join(f"{k[:12]:>12s}" for k in keys))
    for kind, rows in acc.items():
        med = {k: np.nanmedian([r[k] for r in rows]) for k in keys}
        print(f"{kind:6s} " + " ".join(f"{med[k]:12.2f}" for k in keys))


if __name__ == "__main__":
    main(sys.argv[1])


def finalize_split(path):
    """Median (over launches and finalizing CTAs) of: publish+atomic, fold, finalize #1 and,
    in the ICR_DIAG_FIN2 build, the warm repeat of the same finalize (stamp slot 5)."""
    d = np.genfromtxt(path, delimiter=",", names=True)
    out = {}
    for l in sorted(set(int(x) for x in d["launch"])):
        if l == 0 or l >= 193:
            continue
        k = (l - 1) % 6 + 1
        kind = KIND[k if k != 6 else 0]
        if kind in ("attn", "merge"):
            continue
        x = d[(d["launch"] == l) & (d["fin0_done"] >= 0)]
        o = out.setdefault(kind, {"tmem->atomic": [], "atomic->fold": [], "fin1": [], "fin2": []})
        a = x[x["epi_atomic"] >= 0]
        o["tmem->atomic"] += list(a["epi_atomic"] - a["epi_tmem_full"])
        o["atomic->fold"] += list(a["sum_done"] - a["epi_atomic"])
        o["fin1"] += list(x["fin0_done"] - x["sum_done"])
        o["fin2"] += list(x["end"] - x["fin0_done"])
    for kind, o in out.items():
        print(kind, " ".join(f"{k}={np.median(v):.2f}" for k, v in o.items() if v))


if __name__ == "__main__" and len(sys.argv) > 2:
    finalize_split(sys.argv[1])
