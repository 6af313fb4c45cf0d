"""Debug: small engine on a short C4 TFIM prefix (for compute-sanitizer)."""
import math, os, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble
ns, steps = int(sys.argv[1]), int(sys.argv[2])
ham = tb.build_tfim_ring(50, 1.0, 6)
cfg = tb.PaiConfig(math.pi / 2**8, steps, 3.0 * steps / 750)
p = ensemble.pack_ensemble(ham, cfg, 7, range(ns), "0" * 50, tb.TruncationPolicy(16, 1e-12), np.array([steps]))
out = {}
for small in sys.argv[3:]:
    os.environ["TB_SMALL_ENGINE"] = small
    out[small] = ensemble.run_packed(p)
    print("engine small =", small, "ok, kernel ms", out[small].kernel_ms, flush=True)
if len(out) == 2:
    d = np.abs(out["0"].values - out["1"].values)
    print("max diff", d.max(), "samples differing", int((d.max(axis=(1, 2)) > 0).sum()))
