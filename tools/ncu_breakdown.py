"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel:
python tools/ncu_breakdown.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
d = collections.defaultdict(list)
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") == "gpu__time_duration.sum":
            d[rec["Kernel Name"].split("(")[0][:48]].append(float(rec["Metric Value"]))
tot = sum(sum(v) for v in d.values())
print(f"total {tot / 1e3:.1f} us over {sum(len(v) for v in d.values())} launches")
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{sum(v) / 1e3:10.1f} us  {len(v):4d}x  mean {sum(v) / len(v) / 1e3:8.1f} us  "
          f"{100 * sum(v) / tot:5.1f}%  {k}")
