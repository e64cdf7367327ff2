"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr, data = rows[h], rows[h + 1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0].replace("void ", "")[:70]
    agg[name][0] += 1
    agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"{'ms':>9} {'share':>6} {'launches':>8}  kernel   (ncu launch list: cold-cache, serialised)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[1]/1e6:9.3f} {100*v[1]/tot:5.1f}% {v[0]:8d}  {k}")
