"""A/B of the 8-CTA cluster Jacobi (jacobi_cluster) against the single-CTA
wide path (jacobi_wide) on the chi = 128 problems.
  1. tb_svd of 256x256 complex matrices with an MPS-like spectrum: one matrix
     (latency: the sequential-stage case) and a batch (throughput);
  2. the C5 deterministic Trotter stage (N=32 ring, seed 8, chi 128) for the
     first STEPS steps through tb_run_stream, both ways, with <Z_j> compared.
usage: python tools/time_cluster.py [STEPS]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb  # noqa: E402
from paper_2604_13144_b200 import _lib  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 25
lib, ctx = _lib.load(), _lib.context(0)
rng = np.random.default_rng(0)
m = n = 256
sv = np.concatenate([np.logspace(0, -6, 128), np.logspace(-7, -13, 128)])
mats = []
for i in range(18):
    q1, _ = np.linalg.qr(rng.normal(size=(m, m)) + 1j * rng.normal(size=(m, m)))
    q2, _ = np.linalg.qr(rng.normal(size=(n, n)) + 1j * rng.normal(size=(n, n)))
    mats.append((q1 * sv) @ q2.conj().T)
mats = np.ascontiguousarray(np.stack(mats))
for b in (1, 18):
    for cl in ("0", "1"):
        os.environ["TB_CLUSTER"] = cl
        s = np.zeros((b, 256))
        best = 1e9
        for rep in range(3):
            t0 = time.perf_counter()
            _lib.check(lib.tb_svd(ctx, mats.ctypes.data, b, m, n, s.ctypes.data, None, None), ctx)
            best = min(best, time.perf_counter() - t0)
        err = np.max(np.abs(s - sv[None]) / sv[0])
        print(f"svd 256x256 batch {b:2d} cluster={cl}: {best * 1e3:8.2f} ms wall (incl. H2D/D2H), "
              f"max rel sv err {err:.1e}", flush=True)

ham = tb.build_spin_ring(32, 1.0, 8)
pol = tb.TruncationPolicy(128, 1e-12)
res = {}
for cl in ("1", "0"):
    os.environ["TB_CLUSTER"] = cl
    st = tb.init_product_state("01" * 16)
    t0 = time.time()
    done = 0
    while done < steps:
        k = min(5, steps - done)
        tb.run_circuit(st, tb.build_trotter_circuit(ham, k * 2.0 / 200, k), pol)
        done += k
        print(f"  cluster={cl} trotter step {done}: {time.time() - t0:.1f} s, max bond {tb.max_bond(st)}, "
              f"discarded {st.discarded_weight:.3e}", flush=True)
    z = np.array([tb.expectation(st, tb.PauliString.single(32, q, "Z")) for q in range(32)])
    res[cl] = (time.time() - t0, st.bond_dims, st.discarded_weight, z)
    print(f"C5 Trotter stage, {steps} steps, cluster={cl}: {res[cl][0]:.1f} s", flush=True)
if "0" in res:
    print("bond dims equal:", res["0"][1] == res["1"][1], " discarded", res["0"][2], res["1"][2],
          " max |dZ|", float(np.max(np.abs(res["0"][3] - res["1"][3]))), " speed-up", res["0"][0] / res["1"][0])
