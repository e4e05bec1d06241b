"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python profiles/launch_summary.py launches.csv [skip_first_n_launches]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
h = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows:
    if h is None:
        if "Kernel Name" in r:
            h = r
        continue
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum" or int(d["ID"]) < skip:
        continue
    name = d["Kernel Name"].split("(")[0].split("::")[-1]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:40s} n={v[0]:5d} total_us={v[1]:10.1f} mean_us={v[1] / v[0]:8.2f} share={v[1] / tot:.3f}")
