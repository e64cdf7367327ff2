"""Summarise an ncu report: key metrics + stall reasons by SASS opcode."""
import csv, subprocess, sys
from collections import Counter, defaultdict

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.per_cycle_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg"]
for h, u, v in zip(hdr, units, vals):
    if h in want:
        print(f"{h:80s} {v} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; data = rows[2:]
i_src = hdr.index("Source"); i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_ex = hdr.index("Instructions Executed")
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
agg = defaultdict(Counter); cnt = Counter(); tot = 0
for r in data:
    if not r[i_s].isdigit():
        continue
    toks = r[i_src].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    tot += int(r[i_s]); cnt[op] += int(r[i_ex] or 0)
    for c in cols:
        v = r[hdr.index(c)]
        if v.isdigit():
            agg[op][c] += int(v)
print("total samples", tot)
byop = sorted(agg, key=lambda o: -sum(agg[o].values()))
for op in byop[:12]:
    s = sum(agg[op].values())
    top = ", ".join(f"{k[6:]}={v}" for k, v in agg[op].most_common(4))
    print(f"{op:8s} {100*s/tot:5.1f}% exec={cnt[op]:>11d}  {top}")
