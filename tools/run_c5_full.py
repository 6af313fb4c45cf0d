"""Config 5 (hybrid Trotter -> TE-PAI) end to end on one B200, on the REAL t0
state (trotter.py:48-57, mps.py:296-338).

  t0 OUT.mps            deterministic first-order Trotter circuit of the N=32
                        ring (seed 8) from the Neel state to t0 = 2.0 in 200
                        steps at chi 128 (one circuit: tb_run_stream, one CTA),
                        snapshot written in the reference's MPS1 format
  tepai IN.mps N_SAMPLES  TE-PAI extension over a further T = 1.0 (100 steps,
                        Delta = pi/2^7, circuits from seed 9), every sample
                        starting from the snapshot, chi 128, <Z_j> for all j at
                        10 checkpoints; prints the rate, FLOP/s and the SPEC
                        results table for sites 0 and 16.
"""
import math
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb  # noqa: E402
from paper_2604_13144_b200 import ensemble, estimator  # noqa: E402

ham = tb.build_spin_ring(32, 1.0, 8)
pol = tb.TruncationPolicy(128, 1e-12)
mode = sys.argv[1]
if mode == "t0":
    st = tb.init_product_state("01" * 16)
    t0 = time.time()
    for done in range(0, 200, 10):
        tb.run_circuit(st, tb.build_trotter_circuit(ham, 10 * 2.0 / 200, 10), pol)
        print(f"trotter step {done + 10}/200: {time.time() - t0:.1f} s, max bond {tb.max_bond(st)}, "
              f"discarded {st.discarded_weight:.3e}", flush=True)
    tb.save_snapshot(st, sys.argv[2])
    z = [tb.expectation(st, tb.PauliString.single(32, q, "Z")) for q in range(32)]
    print(f"t0 stage done in {time.time() - t0:.1f} s; bonds {st.bond_dims}; <Z_0..3>(t0) = {np.round(z[:4], 6)}")
else:
    st0 = tb.load_snapshot(sys.argv[2])
    ns = int(sys.argv[3])
    cfg = tb.PaiConfig(math.pi / 2**7, 100, 1.0)
    ck = np.arange(10, 101, 10)
    t0 = time.time()
    p = ensemble.pack_ensemble(ham, cfg, 9, range(ns), "01" * 16, pol, ck, init_state=st0)
    tp = time.time() - t0
    r = ensemble.run_packed(p, keep_values=False)
    st = r.stats()
    print(f"C5 TE-PAI stage from the real t0 state (bonds up to {st0.max_bond()}): samples={ns} "
          f"kernel_s={r.kernel_ms / 1e3:.1f} -> {ns / (r.kernel_ms / 1e3):.3f} samples/s, "
          f"TF/s={r.flops / r.kernel_ms / 1e9:.3f}, updates/sample={r.ledger[:, 0].mean():.0f}, "
          f"chi_max={r.ledger[:, 2].max():.0f}, host pack {tp:.1f} s")
    times = 2.0 + ck * 1.0 / 100
    for site in (0, 16):
        print(f"site {site}:")
        print(estimator.results_table(times, st, r.weights, site, mean_nu=float(np.mean(p.nu)),
                                      mean_cost=float(r.ledger[:, 1].mean()), chi_max=int(r.ledger[:, 2].max())),
              end="")
