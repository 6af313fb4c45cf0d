"""Config 4 (TFIM ring) on the GPU: N=50 periodic disordered transverse-field
Ising ring (build_tfim_ring, seed 6), all-|0> start, T=3.0, Delta=pi/2^8,
circuits from seed 7, <Z_j> for all j at 30 checkpoints, chi 16 or 128, plus
the single deterministic Trotter circuit at the same chi on the same kernels.

As written (300 steps) the config is outside the sampler's domain
(max|theta| = 0.0296 > Delta = 0.0123, PaiConfig.validate_against raises), so
the step count is raised to 750 = 30 x 25 (min_trotter_steps gives 725), the
first multiple of the checkpoint count that is accepted.  ``MAX_STEP`` cuts
the circuits to a prefix at the same step size (PaiConfig(delta, MAX_STEP,
3.0 * MAX_STEP / 750)); the rate is reported for the prefix.
usage: python tools/time_c4.py CHI N_SAMPLES MAX_STEP [--trotter]"""
import math, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble

chi, ns, mx = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
n, steps, T = 50, 750, 3.0
ham = tb.build_tfim_ring(n, 1.0, 6)
delta = math.pi / 2**8
assert tb.min_trotter_steps(ham, delta, T) <= steps
cfg = tb.PaiConfig(delta, mx, T * mx / steps)
ck = np.arange(25, mx + 1, 25) if mx >= 25 else np.array([mx])
pol = tb.TruncationPolicy(chi, 1e-12)
t0 = time.time()
p = ensemble.pack_ensemble(ham, cfg, 7, range(ns), "0" * n, pol, ck)
r = ensemble.run_packed(p)
print(f"C4 TFIM chi={chi}: samples={ns} steps={mx}/{steps} kernel_s={r.kernel_ms/1e3:.2f} "
      f"wall_s={time.time()-t0:.1f} updates/sample={r.ledger[:,0].mean():.0f} chi_max={r.ledger[:,2].max():.0f} "
      f"TF/s={r.flops/r.kernel_ms/1e9:.3f} prefix samples/s={ns / (r.kernel_ms / 1e3):.3f}")
print("ensemble mean <Z_0..4> at last checkpoint:", np.round(r.values[:, -1, :5].mean(axis=0) if r.values is not None
                                                             else [], 4))
if "--trotter" in sys.argv:
    st, done, t1 = tb.init_product_state("0" * n), 0, time.time()
    out = []
    for j in ck:
        tb.run_circuit(st, tb.build_trotter_circuit(ham, (j - done) * T / steps, int(j - done)), pol)
        done = int(j)
        out.append([tb.expectation(st, tb.PauliString.single(n, q, "Z")) for q in range(5)])
    print(f"deterministic Trotter chi={chi}: steps={mx} wall_s={time.time()-t1:.1f} max_bond={tb.max_bond(st)} "
          f"discarded={st.discarded_weight:.3e} <Z_0..4>={np.round(out[-1], 4)}")
