"""Time the engine on a prefix of a config's circuits (exploration tool).
usage: python tools/time_prefix.py N_SITES CHI HAM_SEED CIRC_SEED STEPS T N_SAMPLES MAX_STEP"""
import os, sys; sys.path.insert(0, "."); import __graft_entry__  # noqa: E702
# the library path is bound when the package is first imported (inside build()): set it before
os.environ.setdefault("TB_PROFILE", "1"); os.environ.setdefault("TB_LIB", __graft_entry__.LIB_PROF)  # phase counters: diagnostics build
__graft_entry__.build(profile=True)
import math, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import packing, ensemble

n, chi, hs, cs, steps, T, ns, mx = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]),
                                     int(sys.argv[5]), float(sys.argv[6]), int(sys.argv[7]), int(sys.argv[8]))
ham = tb.build_spin_ring(n, 1.0, hs)
cfg = tb.PaiConfig(math.pi / 2**7, steps, T)
ck = np.arange(10, mx + 1, 10)
table = packing.TermTable.of(ham)
t0 = time.time()
ps = [packing.pack_sampled(tb.sample_circuit(ham, cfg, tb.circuit_stream(cs, i), sample_id=i).prefix(mx), table, ck)
      for i in range(ns)]
w, off, ce, sg = packing.pack_batch(ps, ck.size)
t1 = time.time()
p = ensemble.PackedEnsemble(n, min(chi, 2 ** (n // 2)), min(chi, 2 ** (n // 2)), 1e-12, w, off, ce, sg,
                            packing.angle_table(packing.tepai_angles(cfg.delta)),
                            ensemble.checkpoint_weights(ham, cfg, ck), np.arange(n, dtype=np.int32),
                            np.stack([tb.mps.SITE_VECTORS[c] for c in "01" * (n // 2)]).view(np.float64).reshape(n, 4).copy(),
                            np.arange(ns), np.diff(off), True)
r = ensemble.run_packed(p)
print(f"n={n} chi={chi} samples={ns} max_step={mx} gates={w.size} pack_s={t1-t0:.2f} kernel_ms={r.kernel_ms:.1f} "
      f"wall_s={r.wall_s:.2f} flops={r.flops:.3e} TF/s={r.flops/r.kernel_ms/1e9:.3f} "
      f"updates={r.ledger[:,0].sum():.0f} chi3={r.ledger[:,1].sum():.3e} disc={r.ledger[:,3].mean():.2e}")
from paper_2604_13144_b200 import _lib
pr = _lib.debug_profile().astype(np.float64)
tot = pr[7]
print("phase share: jacobi %.3f (qrcp %.3f) qr %.3f gemm+gate %.3f post %.3f measure %.3f | calls %d avg sweeps %.2f | 128x128: calls %d avg sweeps %.2f avg Mcyc %.3f" % (
    pr[0]/tot, pr[12]/tot, pr[3]/tot, pr[4]/tot, pr[5]/tot, pr[6]/tot, pr[1], pr[2]/max(pr[1],1), pr[10], pr[11]/max(pr[10],1), pr[9]/max(pr[10],1)/1e6))
print("qrcp calls %d avg steps %.1f cyc/step %.0f | within %.3f cross %.3f of total" % (
    pr[8], pr[15]/max(pr[8],1), pr[12]/max(pr[15],1), pr[13]/tot, pr[14]/tot))
print("Mw=128 cycles per sweep index (k cycles):", [int(pr[40+k]/max(pr[56+min(k,7)],1)/1e3) for k in range(8)], "counts", pr[56:64].astype(int).tolist())
print("jacobi overheads (share of total): build_l %.3f staging %.3f refresh %.3f swap %.3f writeback %.3f sort_sigma %.3f" % tuple(pr[24:30] / tot))
print("qrcp sub-phases (cycles/step, thread 0 view): pivot %.0f publish %.0f normalise %.0f update %.0f barrier %.0f" % tuple(
    pr[32:37] / max(pr[15], 1)))
print("two-site front end (share of total): theta GEMM %.3f gate pass %.3f" % (pr[30] / tot, pr[31] / tot))
print("gram screen: calls %d, k cycles per call %.0f, share of total %.3f" % (pr[39], pr[38] / max(pr[39], 1) / 1e3, pr[38] / tot))
