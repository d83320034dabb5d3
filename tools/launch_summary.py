"""Summarise an ncu launch list (gpu__time_duration.sum) for the last run of profile_run.py."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
per_run = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[h], rows[h + 1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
ours = [r for r in data if "farqb" in r[ki]]
run = ours[-per_run:] if per_run else ours
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in run:
    name = r[ki].split("(")[0]
    for junk in ("void ", "farqb::", "(anonymous namespace)::", "<unnamed>::"):
        name = name.replace(junk, "")
    us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    agg[name][0] += 1
    agg[name][1] += us
    tot += us
print(f"{len(run)} launches, {tot:.1f} us total (serialised, cold cache)")
for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us:9.1f} us {100 * us / tot:5.1f}%  {c:4d}x  {k[:100]}")
