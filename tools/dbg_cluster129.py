"""Debug: which switch removes the cluster-Jacobi failures?"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_13144_b200 import _lib as engine

def svd_gpu(a):
    lib, ctx = engine.load(), engine.context(0)
    a = np.ascontiguousarray(a, np.complex128)
    b, m, n = a.shape
    k = min(m, n)
    s = np.zeros((b, k)); u = np.zeros((b, m, k), np.complex128); vh = np.zeros((b, k, n), np.complex128)
    engine.check(lib.tb_svd(ctx, a.ctypes.data, b, m, n, s.ctypes.data, u.ctypes.data, vh.ctypes.data), ctx)
    return u, s, vh

def mats(m, n):
    rng = np.random.default_rng(m * 1000 + n)
    k = min(m, n)
    q1, _ = np.linalg.qr(rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k)))
    q2, _ = np.linalg.qr(rng.normal(size=(n, k)) + 1j * rng.normal(size=(n, k)))
    sv = np.logspace(0, -14, k)
    if k >= 8:
        sv[-(k // 8):] = 0.0
    return np.stack([(q1 * sv) @ q2.conj().T, rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))])

def errs(a, u, s, vh):
    out = []
    for b in range(a.shape[0]):
        ref = np.linalg.svd(a[b], compute_uv=False)
        e_s = np.max(np.abs(s[b] - ref)) / ref[0]
        e_r = np.linalg.norm((u[b] * s[b]) @ vh[b] - a[b]) / np.linalg.norm(a[b])
        live = s[b] > 1e-10 * s[b][0]
        uu = u[b][:, live]
        e_o = np.abs(uu.conj().T @ uu - np.eye(uu.shape[1])).max()
        out.append((e_s, e_r, e_o))
    return out

for shape in [(256, 17), (160, 250), (129, 129), (256, 256), (136, 256)]:
    a = mats(*shape)
    for pre in ("0", "1"):
        for dbg in ("0", "1", "2", "3"):
            os.environ.update(TB_CLUSTER="1", TB_PRECOND=pre, TB_CLUSTER_TMA="1", TB_CL_DBG=dbg)
            worst = np.zeros(3); bad = 0
            for rep in range(6):
                e = np.array(errs(a, *svd_gpu(a)))
                worst = np.maximum(worst, e.max(axis=0))
                bad += int(e[:, 0].max() > 1e-13 or e[:, 1].max() > 1e-12 or e[:, 2].max() > 1e-12)
            print(shape, "precond", pre, "dbg", dbg, "(1: no offmax shortcut, 2: no pair skipping)", "bad reps", bad, "/ 6",
                  "worst sv %.1e rec %.1e orth %.1e" % tuple(worst), flush=True)
