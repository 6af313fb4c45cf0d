"""Reference-vs-reference spreads of the truncated regime (CPU only): per
checkpoint, the median and 90th percentile over (sample, site) of
|zgesvd - zgesdd| and of |zgesdd(A^H) - zgesdd(A)| for the samples the third
twin covers (tests/golden/make_golden_trunc.py --third-twin N), next to the
GPU-vs-reference quantiles of a truncated_stats_*.txt table if one is given.
usage: python tools/trunc_twin_spread.py c3 [profiles/r02v_truncated_stats_c3_faithful.txt]"""
import sys
import numpy as np

name = sys.argv[1]
ref = np.load(f"tests/golden/ref_{name}_stat.npz")
tw = np.load(f"tests/golden/ref_{name}_stat_twinT.npz")
n = tw["vals_gesdd_t"].shape[0]
a, b, c = ref["vals_gesdd"][:n], ref["vals_gesvd"][:n], tw["vals_gesdd_t"]
gpu = {}
if len(sys.argv) > 2:
    for line in open(sys.argv[2]):
        if not line.startswith("#"):
            f = line.split()
            gpu[int(f[0])] = (float(f[2]), float(f[5]))
print(f"# {name}: first {n} samples; |gesvd - gesdd| and |gesdd(A^H) - gesdd(A)| (50% / 90%), GPU-vs-reference (64 samples)")
print("# ckpt  gesvd50 gesvd90   transp50 transp90   gpu50 gpu90   gpu50/transp50 gpu90/transp90")
for k in range(a.shape[1]):
    d1, d2 = np.abs(b[:, k] - a[:, k]).ravel(), np.abs(c[:, k] - a[:, k]).ravel()
    q = [np.percentile(d1, 50), np.percentile(d1, 90), np.percentile(d2, 50), np.percentile(d2, 90)]
    g = gpu.get(k)
    tail = "  %.3e %.3e   %.2f %.2f" % (g[0], g[1], g[0] / max(q[2], 1e-300), g[1] / max(q[3], 1e-300)) if g else ""
    print("%2d  %.3e %.3e   %.3e %.3e%s" % (k, q[0], q[1], q[2], q[3], tail))
