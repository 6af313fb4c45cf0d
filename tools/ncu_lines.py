"""Per-CUDA-source-line stall samples / executed instructions from an ncu report."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hi]
S, E = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
def num(x):
    try: return float(x)
    except ValueError: return 0.0
agg, cur, src = {}, None, {}
for r in rows[hi + 1:]:
    if len(r) < len(hdr): continue
    if r[0]:
        if r[0].isdigit():
            cur = int(r[0]); src[cur] = r[1]
        continue
    if cur is None: continue
    a = agg.setdefault(cur, [0.0, 0.0]); a[0] += num(r[S]); a[1] += num(r[E])
ts = sum(v[0] for v in agg.values()); te = sum(v[1] for v in agg.values())
for ln, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]/ts:6.3f} {v[1]/te:6.3f} L{ln:>5}: {src.get(ln,'').strip()[:95]}")
