"""Hot regions of an ncu report: SASS grouped into runs between barriers /
branches, with samples, top stall reasons and instruction mix per run.
python tools/ncu_hot.py rep.ncu-rep [min_pct]"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]; minpct = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; data = rows[2:]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_ex = hdr.index("Instructions Executed")
cols = [(c, hdr.index(c)) for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[i_s]) for r in data if r[i_s].isdigit())
runs = []; cur = None
def op_of(s):
    t = s.split()
    if not t: return ""
    return (t[1] if t[0].startswith("@") and len(t) > 1 else t[0]).split(".")[0]
for idx, r in enumerate(data):
    if not r[i_s].isdigit(): continue
    op = op_of(r[i_src])
    if cur is None:
        cur = dict(start=idx, n=0, samples=0, st=Counter(), ops=Counter(), ex=0)
    cur["n"] += 1; cur["samples"] += int(r[i_s]); cur["ops"][op] += 1
    cur["ex"] = max(cur["ex"], int(r[i_ex] or 0))
    for c, i in cols:
        if r[i].isdigit(): cur["st"][c[6:]] += int(r[i])
    if op in ("BAR", "BRA", "EXIT", "BSYNC", "RET", "CALL", "WARPSYNC"):
        cur["end"] = idx; runs.append(cur); cur = None
if cur: cur["end"] = len(data) - 1; runs.append(cur)
print(f"total samples {tot}, {len(runs)} runs")
for r in sorted(runs, key=lambda x: -x["samples"]):
    p = 100 * r["samples"] / tot
    if p < minpct: break
    ops = ", ".join(f"{k}:{v}" for k, v in r["ops"].most_common(6))
    st = ", ".join(f"{k}={v}" for k, v in r["st"].most_common(5))
    print(f"{p:5.1f}%  rows {r['start']}-{r['end']} ({r['n']} instr, exec {r['ex']})  [{ops}]  {st}")
