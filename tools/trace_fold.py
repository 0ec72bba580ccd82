"""Per split tile of each GEMM launch in a step trace (tools/trace_step.py CSV): when the
finalizer's accumulator was ready, when its last publisher published, when the fold and the
finalize completed (us after the launch's median griddepcontrol.wait return).

  python tools/trace_fold.py gpurun_out/trace.csv
"""
import sys

import numpy as np

KIND = {1: "qkv", 2: "attn", 3: "merge", 4: "o", 5: "gu", 0: "down"}
SHAPE = {"qkv": (6144, 4096, 2), "o": (4096, 4096, 2), "gu": (28672, 4096, 4), "down": (4096, 14336, 2)}


def main(path, G=148):
    d = np.genfromtxt(path, delimiter=",", names=True)
    out = {}
    for l in sorted(set(int(x) for x in d["launch"])):
        if l == 0 or l >= 193:
            continue
        k = (l - 1) % 6 + 1
        kind = KIND[k if k != 6 else 0]
        if kind not in SHAPE:
            continue
        M, K, Lc = SHAPE[kind]
        Ut = K // 64 + Lc
        U = (M // 128) * Ut
        ub = lambda c: (c * U) // G  # noqa: E731
        owner = lambda x: ((x + 1) * G - 1) // U  # noqa: E731
        x = d[d["launch"] == l]
        by = {int(r["cta"]): r for r in x}
        pd = np.median(x["prev_done"])
        for t in range(M // 128):
            cf, cl = owner(t * Ut), owner(t * Ut + Ut - 1)
            if cl == cf or cf not in by:
                continue
            f = by[cf]
            pub = max(by[c]["epi_atomic"] for c in range(cf + 1, cl + 1))
            out.setdefault(kind, []).append([cl - cf + 1, f["epi_tmem_full"] - pd, pub - pd,
                                             f["sum_done"] - pd, f["end"] - pd, f["fin0_done"] - pd])
    print("kind  nseg  tmem_ready  last_pub  fold_done  rearm_done fin_done   (medians; worst tile by fin_done)")
    for kind, v in out.items():
        v = np.array(v)
        w = v[np.argmax(v[:, 5])]
        print(f"{kind:5s} " + " ".join(f"{a:9.2f}" for a in np.median(v, axis=0)) + "  | worst " +
              " ".join(f"{a:7.2f}" for a in w))


if __name__ == "__main__":
    main(sys.argv[1])
