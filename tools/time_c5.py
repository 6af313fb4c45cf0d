"""Time the C5 TE-PAI stage (N=32, chi=128, seed 8/9) on a saturated start MPS.
The t0 = 2.0 Trotter state is replaced by a random mixed-canonical MPS with the
saturated bond profile (1,2,4,...,128,...,128,...,4,2,1): every two-site update
then has the 256 x 256 shape of the real run; the <Z_j> values are meaningless.
The circuits are the C5 TE-PAI stage cut to MAX_STEP Trotter steps at the same
step size (PaiConfig(delta, MAX_STEP, MAX_STEP / 100)): identical per-step
angles and gate statistics, so the rate extrapolates linearly to 100 steps.
usage: python tools/time_c5.py N_SAMPLES MAX_STEP [N_SITES]"""
import os, sys; sys.path.insert(0, "."); import __graft_entry__  # noqa: E702
# the library path is bound when the package is first imported (inside build()): set it before
os.environ.setdefault("TB_PROFILE", "1"); os.environ.setdefault("TB_LIB", __graft_entry__.LIB_PROF)  # phase counters: diagnostics build
__graft_entry__.build(profile=True)
import math, sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble

ns, mx = int(sys.argv[1]), int(sys.argv[2])
NSITES = int(sys.argv[3]) if len(sys.argv) > 3 else 32
n, chi = NSITES, 128
ham = tb.build_spin_ring(n, 1.0, 8)
cfg = tb.PaiConfig(math.pi / 2**7, mx, mx / 100.0)
rng = np.random.default_rng(0)
dims = np.array([min(2 ** min(b, n - b), chi) for b in range(n + 1)], np.int64)
st = tb.MPSState(n)
st.ensure_capacity(chi)
st.dims[:] = dims
for s in range(n - 1, 0, -1):  # right-canonical sites 1..n-1 (rows orthonormal)
    cl, cr = dims[s], dims[s + 1]
    m = rng.normal(size=(cl, 2 * cr)) + 1j * rng.normal(size=(cl, 2 * cr))
    q, _ = np.linalg.qr(m.conj().T)
    st.buf[s, :cl, :, :cr] = q.conj().T[:cl].reshape(cl, 2, cr)
v = rng.normal(size=(1, 2, dims[1])) + 1j * rng.normal(size=(1, 2, dims[1]))
st.buf[0, :1, :, :dims[1]] = v / np.linalg.norm(v)
st.center = 0
ck = np.arange(10, mx + 1, 10) if mx >= 10 else np.array([mx])
t0 = time.time()
p = ensemble.pack_ensemble(ham, cfg, 9, range(ns), "01" * (n // 2), tb.TruncationPolicy(chi, 1e-12), ck, init_state=st)
r = ensemble.run_packed(p)
print(f"C5 TE-PAI stage: samples={ns} steps={mx} kernel_s={r.kernel_ms/1e3:.1f} wall_s={time.time()-t0:.1f} "
      f"updates/sample={r.ledger[:,0].mean():.0f} chi_max={r.ledger[:,2].max():.0f} TF/s={r.flops/r.kernel_ms/1e9:.3f} "
      f"-> {ns / (r.kernel_ms / 1e3) * mx / 100:.4f} full-circuit samples/s (linear extrapolation)")
from paper_2604_13144_b200 import _lib
pr = _lib.debug_profile().astype(np.float64)
tot = pr[7]
print("phase share: jacobi %.3f (qrcp %.3f, within %.3f, cross %.3f) moves %.3f gemm %.3f gate %.3f post %.3f | "
      "svd calls %d avg sweeps %.2f qrcp avg steps %.1f" % (
          pr[0] / tot, pr[12] / tot, pr[13] / tot, pr[14] / tot, pr[3] / tot, pr[30] / tot, pr[31] / tot, pr[5] / tot,
          pr[1], pr[2] / max(pr[1], 1), pr[15] / max(pr[8], 1)))
