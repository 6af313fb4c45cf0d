"""Batched 128x128 complex SVD through tb_svd (one CTA per matrix) — the
Jacobi kernel in isolation, for timing and ncu.  usage: prof_svd.py [batch] [reps] [m] [n]"""
import os, sys; sys.path.insert(0, "."); import __graft_entry__  # noqa: E702
# the library path is bound when the package is first imported (inside build()): set it before
os.environ.setdefault("TB_PROFILE", "1"); os.environ.setdefault("TB_LIB", __graft_entry__.LIB_PROF)  # phase counters: diagnostics build
__graft_entry__.build(profile=True)
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2604_13144_b200 import _lib

b = int(sys.argv[1]) if len(sys.argv) > 1 else 148
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = int(sys.argv[3]) if len(sys.argv) > 3 else 128
n = int(sys.argv[4]) if len(sys.argv) > 4 else 128
rng = np.random.default_rng(0)
k = min(m, n)
# MPS-like spectrum: geometric decay to 1e-6 over the first half, tiny tail
sv = np.concatenate([np.logspace(0, -6, k // 2), np.logspace(-7, -13, k - k // 2)])
a = np.empty((b, m, n), np.complex128)
for i in range(b):
    q1, _ = np.linalg.qr(rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k)))
    q2, _ = np.linalg.qr(rng.normal(size=(n, k)) + 1j * rng.normal(size=(n, k)))
    a[i] = (q1 * sv) @ q2.conj().T
lib, ctx = _lib.load(), _lib.context(0)
s = np.zeros((b, k))
for r in range(reps):
    t0 = time.perf_counter()
    _lib.check(lib.tb_svd(ctx, a.ctypes.data, b, m, n, s.ctypes.data, None, None), ctx)
    dt = time.perf_counter() - t0
    print(f"batch {b} {m}x{n}: {dt*1e3:.1f} ms wall ({dt/b*1e3*148:.2f} ms per SM-SVD if 148 concurrent), "
          f"max rel sv err {np.max(np.abs(s[0]-sv)/sv[0]):.2e}")
pr = _lib.debug_profile().astype(np.int64)
print("svd calls", pr[1], "avg sweeps", pr[2] / max(pr[1], 1), "rotations per sweep (summed):", pr[16:16 + 24].tolist())
# well-conditioned random matrices
a2 = (rng.normal(size=(b, m, n)) + 1j * rng.normal(size=(b, m, n)))
_lib.check(lib.tb_svd(ctx, a2.ctypes.data, b, m, n, s.ctypes.data, None, None), ctx)
pr = _lib.debug_profile().astype(np.int64)
ref = np.linalg.svd(a2[0], compute_uv=False)
print("random: avg sweeps", pr[2] / max(pr[1], 1), "rot/sweep:", pr[16:16 + 24].tolist(), "err", np.max(np.abs(s[0]-ref))/ref[0])
