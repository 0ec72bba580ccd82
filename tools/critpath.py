"""Critical path of a traced decode step: per kernel kind, the time from its predecessor's
completion (its own griddepcontrol.wait return) to its successor's wait return."""
import sys
import numpy as np
d = np.genfromtxt(sys.argv[1], delimiter=",", names=True)
kinds = {1: "qkv", 2: "attn", 3: "merge", 4: "o", 5: "gu", 0: "down"}
prev = {}
for l in sorted(set(int(x) for x in d["launch"])):
    x = d[d["launch"] == l]
    pd = x["prev_done"][x["prev_done"] >= 0]
    prev[l] = np.median(pd) if len(pd) else np.nan
ls = sorted(prev)
acc = {k: [] for k in kinds.values()}
for a, b in zip(ls, ls[1:]):
    if 1 <= a < 193 and b == a + 1:
        acc[kinds[(a - 1) % 6 + 1 if (a - 1) % 6 + 1 != 6 else 0]].append(prev[b] - prev[a])
tot = 0
for k, v in acc.items():
    if v:
        tot += np.median(v)
        print(f"{k:6s} critical {np.median(v):7.2f} us  (min {np.min(v):6.2f} max {np.max(v):6.2f})")
print(f"sum per layer {tot:.1f} us")
