"""Run-to-run bitwise determinism of the ensemble engine on a config prefix,
for both engines (TB_SMALL_ENGINE=0/1 where the capacity allows it).
usage: python tools/check_determinism.py"""
import math, os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble

d8 = math.pi / 2**8
cases = [("C4 TFIM N=50 chi=16, 100 steps", tb.build_tfim_ring(50, 1.0, 6), tb.PaiConfig(d8, 100, 3.0 * 100 / 750), 7, 592,
          "0" * 50, 16, np.arange(25, 101, 25)),
         ("C2 N=16 chi=32, 60 steps", tb.build_spin_ring(16, 1.0, 2), tb.PaiConfig(math.pi / 2**7, 60, 0.6), 3, 592, "01" * 8,
          32, np.arange(10, 61, 10))]
for name, ham, cfg, seed, ns, labels, chi, ck in cases:
    p = ensemble.pack_ensemble(ham, cfg, seed, range(ns), labels, tb.TruncationPolicy(chi, 1e-12), ck)
    runs = {}
    for small in ("0", "1"):
        os.environ["TB_SMALL_ENGINE"] = small
        runs[small] = [ensemble.run_packed(p) for _ in range(3)]
        for k in (1, 2):
            a, b = runs[small][0], runs[small][k]
            diff = np.abs(a.values - b.values)
            bad = np.argwhere(diff.max(axis=(1, 2)) > 0).ravel()
            print(f"{name}: engine small={small} run 0 vs {k}: identical={np.array_equal(a.values, b.values)} "
                  f"max diff {diff.max():.3e} samples differing {bad.size} first {bad[:8].tolist()} "
                  f"ledger equal {np.array_equal(a.ledger, b.ledger)}", flush=True)
    a, b = runs["0"][0], runs["1"][0]
    diff = np.abs(a.values - b.values)
    bad = np.argwhere(diff.max(axis=(1, 2)) > 0).ravel()
    print(f"{name}: full vs small engine: identical={np.array_equal(a.values, b.values)} max diff {diff.max():.3e} "
          f"samples differing {bad.size} first {bad[:8].tolist()}; first differing checkpoint per sample "
          f"{[int(np.argmax(diff[s].max(axis=1) > 0)) for s in bad[:8]]} discarded there "
          f"{[float(a.discarded[s, int(np.argmax(diff[s].max(axis=1) > 0))]) for s in bad[:4]]}", flush=True)
