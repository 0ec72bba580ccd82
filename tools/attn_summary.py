import json, sys
for f in sys.argv[1:]:
    d = json.load(open(f))
    print(f)
    for r in d["results"]:
        print(f"  ctx {r['context']:6d} adapters {r['adapters']}  {r['ms']*1e3:7.1f} us  {r['gbs']:6.0f} GB/s  {r['frac_of_measured_hbm']:.3f}  items {r['items']}")
