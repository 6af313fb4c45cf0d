import sys, numpy as np
sys.path.insert(0, ".")
from paper_2604_13144_b200 import _lib
lib, ctx = _lib.load(), _lib.context(0)
rng = np.random.default_rng(1)
out = []
for m in (256, 200):
    for n in list(range(33, 41)) + [62, 63, 64, 65, 66, 67, 96, 97, 98]:
        b = 2
        a = (rng.normal(size=(b, m, n)) + 1j * rng.normal(size=(b, m, n))).astype(np.complex128)
        k = min(m, n)
        s = np.zeros((b, k))
        rc = lib.tb_svd(ctx, a.ctypes.data, b, m, n, s.ctypes.data, None, None)
        ref = np.linalg.svd(a, compute_uv=False)
        nb = (n + 31) // 32
        ncl = [n // nb + (1 if bb >= nb - n % nb else 0) for bb in range(nb)]
        out.append(f"{m}x{n} {ncl} err {np.max(np.abs(s - ref) / ref[:, :1]):.1e}")
print("\n".join(out))
