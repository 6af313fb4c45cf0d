"""A/B of the small-problem engine (two resident CTAs per SM, bond capacity
<= 32; TB_SMALL_ENGINE=1, the default) against the full engine (one CTA per SM;
TB_SMALL_ENGINE=0) on the small-chi configs.  Same algorithm and operation
order in both; the two are separate compilations, so values agree to rounding.
usage: python tools/ab_small_engine.py [C1_SAMPLES] [C2_SAMPLES] [C2_STEPS] [C4_SAMPLES] [C4_STEPS]"""
import math, os, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble

a = [int(x) for x in sys.argv[1:]] + [None] * 5
n1, n2, s2, n4, s4 = a[0] or 1000, a[1] or 592, a[2] or 60, a[3] or 592, a[4] or 100
d7, d8 = math.pi / 2**7, math.pi / 2**8
cases = [
    ("C1 N=8 chi=16 full circuits", tb.build_spin_ring(8, 1.0, 0), tb.PaiConfig(d7, 100, 1.0), 1, n1, "01" * 4, 16,
     np.arange(10, 101, 10)),
    (f"C2 N=16 chi=32 first {s2} of 200 steps", tb.build_spin_ring(16, 1.0, 2), tb.PaiConfig(d7, s2, 2.0 * s2 / 200), 3,
     n2, "01" * 8, 32, np.arange(10, s2 + 1, 10)),
    (f"C4 TFIM N=50 chi=16 first {s4} of 750 steps", tb.build_tfim_ring(50, 1.0, 6), tb.PaiConfig(d8, s4, 3.0 * s4 / 750),
     7, n4, "0" * 50, 16, np.arange(25, s4 + 1, 25)),
]
for name, ham, cfg, seed, ns, labels, chi, ck in cases:
    p = ensemble.pack_ensemble(ham, cfg, seed, range(ns), labels, tb.TruncationPolicy(chi, 1e-12), ck)
    res = {}
    for small in ("0", "1"):
        os.environ["TB_SMALL_ENGINE"] = small
        best = None
        for rep in range(2):
            r = ensemble.run_packed(p)
            best = r if best is None or r.kernel_ms < best.kernel_ms else best
        res[small] = best
        print(f"{name}: TB_SMALL_ENGINE={small} samples={ns} kernel_ms={best.kernel_ms:.1f} "
              f"-> {ns / (best.kernel_ms / 1e3):.2f} samples/s, TF/s={best.flops / best.kernel_ms / 1e9:.3f}", flush=True)
    same = np.array_equal(res["0"].values, res["1"].values) and np.array_equal(res["0"].sum_v, res["1"].sum_v)
    worst = float(np.abs(res["0"].values - res["1"].values).max())
    print(f"{name}: speed-up {res['0'].kernel_ms / res['1'].kernel_ms:.3f}x, values bit-identical: {same}, "
          f"max |difference| {worst:.2e}", flush=True)
