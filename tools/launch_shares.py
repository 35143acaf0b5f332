#!/usr/bin/env python3
"""Per-kernel time shares of ncu launch lists (gpu__time_duration.sum) for
profiles/: python tools/launch_shares.py OUT.json NAME=CSV [NAME=CSV ...]"""
import collections
import csv
import json
import sys


def shares(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ik, im, iv, iu = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].replace("void ", "").replace("<unnamed>::", "").replace("unnamed>::", "")
        name = name.replace("r1::", "")
        if name.startswith("at::"):  # torch's own kernels (input generation in the probes)
            continue
        v = float(r[iv].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[iu], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for k, v in agg.items() if "gen_kernel" not in k)
    return {k: {"launches": v[0], "total_us": round(v[1], 1), "share": round(v[1] / tot, 4)}
            for k, v in sorted(agg.items(), key=lambda t: -t[1][1]) if "gen_kernel" not in k}


out = {}
for arg in sys.argv[2:]:
    name, path = arg.split("=", 1)
    out[name] = {"source": path, "kernels": shares(path)}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1)[:2500])
