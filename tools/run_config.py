"""Run a whole BASELINE config ensemble on one GPU (queue mode, tb_run_ensemble)
and print its rate and the SPEC.md:463 results table for one site.
  C1: N=8 ring (seed 0), T=1.0 in 100 steps, 1,000 circuits (seed 1), chi 16, <Z_0> at t=0.1..1.0
  C2: N=16 ring (seed 2), T=2.0 in 200 steps, 10^4 circuits (seed 3), chi 32, <Z_j> at 20 checkpoints
usage: python tools/run_config.py C1|C2 [N_SAMPLES] [BATCH]"""
import math, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble, estimator

CFG = {"C1": dict(n=8, hs=0, cs=1, steps=100, T=1.0, ns=1000, chi=16, every=10),
       "C2": dict(n=16, hs=2, cs=3, steps=200, T=2.0, ns=10000, chi=32, every=10)}
c = CFG[sys.argv[1]]
ns = int(sys.argv[2]) if len(sys.argv) > 2 else c["ns"]
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 2960
ham = tb.build_spin_ring(c["n"], 1.0, c["hs"])
cfg = tb.PaiConfig(math.pi / 2**7, c["steps"], c["T"])
ck = np.arange(c["every"], c["steps"] + 1, c["every"])
pol = tb.TruncationPolicy(c["chi"], 1e-12)
runs, t0, pack_s = [], time.time(), 0.0
for lo in range(0, ns, batch):
    tp = time.time()
    p = ensemble.pack_ensemble(ham, cfg, c["cs"], range(lo, min(ns, lo + batch)), "01" * (c["n"] // 2), pol, ck)
    pack_s += time.time() - tp
    runs.append(ensemble.run_packed(p, keep_values=False))
wall = time.time() - t0
kms = sum(r.kernel_ms for r in runs)
sv = sum(r.sum_v for r in runs)
sv2 = sum(r.sum_v2 for r in runs)
st = estimator.aggregate_fixed(sv, sv2, ns, runs[0].weights)
st["estimate"] = st.get("estimate", st.get("mean"))
flops = sum(r.flops for r in runs)
print(f"{sys.argv[1]}: samples={ns} kernel_s={kms/1e3:.2f} -> {ns/(kms/1e3):.1f} samples/s (kernel), "
      f"{ns/wall:.1f} samples/s incl. host sampling+packing ({pack_s:.1f} s, single thread); TF/s={flops/kms/1e9:.3f}")
print(estimator.results_table(ck * c["T"] / c["steps"], st, runs[0].weights, 0), end="")
