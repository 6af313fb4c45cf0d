"""Config 4 (TFIM ring, N=50) to the END of its 750-step circuits at chi 128
or 16, with the single deterministic Trotter circuit at
the same chi on the same kernels for comparison.  The config's own 300 steps
are outside the sampler's domain, so it runs 750 = 30 x 25.
usage: python tools/run_c4_full.py CHI N_SAMPLES [--trotter-only|--ensemble-only]"""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb  # noqa: E402
from paper_2604_13144_b200 import ensemble, estimator  # noqa: E402

chi, ns = int(sys.argv[1]), int(sys.argv[2])
n, steps, T = 50, 750, 3.0
ham = tb.build_tfim_ring(n, 1.0, 6)
delta = math.pi / 2**8
cfg = tb.PaiConfig(delta, steps, T)
ck = np.arange(25, steps + 1, 25)
pol = tb.TruncationPolicy(chi, 1e-12)
times = ck * T / steps
if "--trotter-only" not in sys.argv:
    t0 = time.time()
    p = ensemble.pack_ensemble(ham, cfg, 7, range(ns), "0" * n, pol, ck)
    r = ensemble.run_packed(p, keep_values=True)
    st = r.stats()
    print(f"C4 TFIM chi={chi}: samples={ns} steps={steps} kernel_s={r.kernel_ms / 1e3:.1f} "
          f"-> {ns / (r.kernel_ms / 1e3):.3f} samples/s, TF/s={r.flops / r.kernel_ms / 1e9:.3f}, "
          f"updates/sample={r.ledger[:, 0].mean():.0f}, chi_max={r.ledger[:, 2].max():.0f}, "
          f"mean discarded={r.ledger[:, 3].mean():.3e}, wall {time.time() - t0:.1f} s", flush=True)
    print("site 0:")
    print(estimator.results_table(times, st, r.weights, 0, mean_nu=float(np.mean(p.nu)),
                                  mean_cost=float(r.ledger[:, 1].mean()), chi_max=int(r.ledger[:, 2].max())), end="")
    np.save(f"gpurun_out/c4_chi{chi}_estimate.npy", st["estimate"])
if "--ensemble-only" not in sys.argv:
    stt, done, t1 = tb.init_product_state("0" * n), 0, time.time()
    out = []
    for j in ck:
        tb.run_circuit(stt, tb.build_trotter_circuit(ham, (j - done) * T / steps, int(j - done)), pol)
        done = int(j)
        out.append([tb.expectation(stt, tb.PauliString.single(n, q, "Z")) for q in range(n)])
        print(f"trotter step {j}: {time.time() - t1:.1f} s, max bond {tb.max_bond(stt)}, "
              f"discarded {stt.discarded_weight:.3e}", flush=True)
    out = np.array(out)
    np.save(f"gpurun_out/c4_chi{chi}_trotter.npy", out)
    print(f"deterministic Trotter chi={chi}: {steps} steps in {time.time() - t1:.1f} s, <Z_0..4>(T) = "
          f"{np.round(out[-1, :5], 4)}")
