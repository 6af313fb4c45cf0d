"""Timing + phase counters of the wide (256-row) SVD path (diagnostic)."""
import os, sys; sys.path.insert(0, "."); import __graft_entry__  # noqa: E702
# the library path is bound when the package is first imported (inside build()): set it before
os.environ.setdefault("TB_PROFILE", "1"); os.environ.setdefault("TB_LIB", __graft_entry__.LIB_PROF)  # phase counters: diagnostics build
__graft_entry__.build(profile=True)
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2604_13144_b200 import _lib
exec(open("tools/prof_svd.py").read().split("lib, ctx")[0])
lib, ctx = _lib.load(), _lib.context(0)
s = np.zeros((b, min(m, n)))
for rep in range(int(sys.argv[5]) if len(sys.argv) > 5 else 4):
    t0 = time.perf_counter()
    _lib.check(lib.tb_svd(ctx, a.ctypes.data, b, m, n, s.ctypes.data, None, None), ctx)
    dt = time.perf_counter() - t0
    pr = _lib.debug_profile().astype(np.float64)
    print(f"rep {rep}: {dt*1e3:.1f} ms  sweeps {pr[2]/max(pr[1],1):.2f}  qrcp Mcyc/call {pr[12]/max(pr[8],1)/1e6:.2f} "
          f"steps {pr[15]/max(pr[8],1):.0f}  err {np.max(np.abs(s[0]-sv)/sv[0]):.1e}")
