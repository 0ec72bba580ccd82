"""Summarise ncu captures into profiles/ (run here, on the CPU box, after a gpurun).

  python tools/summarize_ncu.py <report.ncu-rep> <algorithmic_bytes_per_launch> <out.json>
  python tools/summarize_ncu.py --launches <launches.csv> <out.txt>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_bytes.sum",
        "lts__t_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        res.append({"kernel": d.get("Kernel Name", "")[:120],
                    "metrics": {k: {"value": d[k], "unit": u.get(k, "")} for k in KEYS if k in d}})
    return res


def to_bytes(m):
    v = float(m["value"].replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(m["unit"], 1)


def main():
    if sys.argv[1] == "--launches":
        rows = list(csv.reader(open(sys.argv[2])))
        hdr = None
        agg = defaultdict(lambda: [0, 0.0])
        total = 0.0
        for r in rows:
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                d = dict(zip(hdr, r))
                v = float(d["Metric Value"].replace(",", ""))
                name = d["Kernel Name"].split("(")[0]
                agg[name][0] += 1
                agg[name][1] += v
                total += v
        with open(sys.argv[3], "w") as f:
            f.write("ncu --metrics gpu__time_duration.sum --clock-control none, one C2 decode step "
                    "(tools/profile_step.py step): serialised, cold-cache launch times -- compare shares\n")
            for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
                f.write(f"{c:5d} launches {v / 1e3:9.1f} us {100 * v / total:5.1f}%  avg {v / c / 1e3:7.2f} us  {n}\n")
            f.write(f"total {total / 1e6:.3f} ms over {sum(c for c, _ in agg.values())} launches\n")
        return
    rep, algo, out = sys.argv[1], float(sys.argv[2]), sys.argv[3]
    res = raw(rep)
    for r in res:
        m = r["metrics"]
        if "dram__bytes_read.sum" in m:
            tb = to_bytes(m["dram__bytes_read.sum"]) + to_bytes(m["dram__bytes_write.sum"])
            r["dram_bytes_per_launch"] = tb
            r["algorithmic_bytes_per_launch"] = algo
            r["traffic_over_algorithmic"] = tb / algo if algo else None
    json.dump({"report": rep, "kernels": res, "dram_bytes_per_launch": res[0].get("dram_bytes_per_launch")},
              open(out, "w"), indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    main()
