"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][:70]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'ms':>10} {'share':>6} {'launches':>8} {'avg us':>10}  kernel")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v[1] / 1e3:10.2f} {100 * v[1] / tot:5.1f}% {v[0]:8d} {v[1] / v[0]:10.1f}  {k}")
print(f"{tot / 1e3:10.2f} total ms (serialised, cold-cache ncu replay)")
