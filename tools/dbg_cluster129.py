"""Debug: where does the cluster SVD of the graded 129x129 matrix lose orthogonality?"""
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

def mat(m, n):
    rng = np.random.default_rng(m * 1000 + n)
    k = min(m, n)
    q1, _ = np.linalg.qr(rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k)))
    q2, _ = np.linalg.qr(rng.normal(size=(n, k)) + 1j * rng.normal(size=(n, k)))
    sv = np.logspace(0, -14, k)
    if k >= 8:
        sv[-(k // 8):] = 0.0
    return np.stack([(q1 * sv) @ q2.conj().T])

for shape in [(129, 129), (129, 129), (136, 256), (256, 256)]:
    a = mat(*shape)
    for env in [dict(TB_CLUSTER="1", TB_PRECOND="1", TB_CLUSTER_TMA="1"), dict(TB_CLUSTER="1", TB_PRECOND="1", TB_CLUSTER_TMA="0"),
                dict(TB_CLUSTER="0", TB_PRECOND="1"), dict(TB_CLUSTER="1", TB_PRECOND="0", TB_CLUSTER_TMA="1")]:
        for k in ("TB_CLUSTER", "TB_PRECOND", "TB_CLUSTER_TMA"):
            os.environ.pop(k, None)
        os.environ.update(env)
        for rep in range(12):
            u, s, vh = svd_gpu(a)
            live = s[0] > 1e-10 * s[0][0]
            uu = u[0][:, live]
            g = np.abs(uu.conj().T @ uu - np.eye(uu.shape[1]))
            i, j = np.unravel_index(np.argmax(g), g.shape)
            big = np.argwhere(g > 1e-12)
            if rep < 1 or g.max() > 1e-12:
              print(shape, env, "rep", rep, "max", g.max(), "at", (i, j), "sig", s[0][i] / s[0][0], s[0][j] / s[0][0],
                  "n>1e-12:", len(big), "first:", big[:6].tolist(), flush=True)
        print(shape, env, "done 12 reps", flush=True)
