"""Summarise an ncu report (SOL, scheduler, instruction mix, stall reasons) for profiles/."""
import csv, io, subprocess, sys
from collections import Counter

rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
want = {"Duration", "Elapsed Cycles", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Achieved Occupancy",
        "Eligible Warps Per Scheduler", "No Eligible", "Executed Instructions", "L2 Hit Rate", "L1/TEX Hit Rate"}
for row in det[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:32s} {d['Metric Value']} {d['Metric Unit']}")
rows = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
hdr = rows[1]; ix = {k: i for i, k in enumerate(hdr)}
def num(x):
    try: return float(x)
    except ValueError: return 0.0
ex = Counter(); st = Counter(); reasons = Counter()
for r in rows[2:]:
    if len(r) < len(hdr): continue
    t = r[ix["Source"]].split()
    if not t: continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    ex[op] += num(r[ix["Instructions Executed"]]); st[op] += num(r[ix["Warp Stall Sampling (All Samples)"]])
    for k in hdr:
        if k.startswith("stall_") and "Not Issued" not in k: reasons[k] += num(r[ix[k]])
te, ts = sum(ex.values()), sum(st.values())
print("instruction mix (share of executed | share of stall samples):")
for op, v in ex.most_common(16): print(f"  {op:10s} {v/te:6.3f} | {st[op]/ts:6.3f}")
print("stall reasons:", {k[6:]: round(v/ts, 3) for k, v in reasons.most_common(8)})
