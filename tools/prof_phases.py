"""Cycle breakdown of the batched 128x128 SVD kernel (diagnostic counters)."""
import os, sys; sys.path.insert(0, "."); import __graft_entry__  # noqa: E702
# the library path is bound when the package is first imported (inside build()): set it before
os.environ.setdefault("TB_PROFILE", "1"); os.environ.setdefault("TB_LIB", __graft_entry__.LIB_PROF)  # phase counters: diagnostics build
__graft_entry__.build(profile=True)
import sys, numpy as np
sys.path.insert(0, ".")
from paper_2604_13144_b200 import _lib
exec(open("tools/prof_svd.py").read().split("lib, ctx")[0])  # build matrices a (graded)
lib, ctx = _lib.load(), _lib.context(0)
s = np.zeros((b, min(m, n)))
for rep in range(2):
    rc = lib.tb_svd(ctx, a.ctypes.data, b, m, n, s.ctypes.data, None, None)
    if rc:
        print("tb_svd rc", rc, "(diagnostic run continues)")
pr = _lib.debug_profile().astype(np.float64)
calls = max(pr[1], 1)
print(f"per SVD: sweeps {pr[2]/calls:.2f}  qrcp calls {pr[8]:.0f} qrcp Mcyc {pr[12]/max(pr[8],1)/1e6:.3f} (steps {pr[15]/max(pr[8],1):.1f}, "
      f"{pr[12]/max(pr[15],1):.0f} cyc/step)  within Mcyc {pr[13]/calls/1e6:.3f}  cross Mcyc {pr[14]/calls/1e6:.3f}  "
      f"per sweep: within {pr[13]/pr[2]/1e3:.1f}k cross {pr[14]/pr[2]/1e3:.1f}k")
st = max(pr[15], 1)
print("qrcp per step (thread 0 view): pivot %.0f owner %.0f bar1 %.0f update %.0f bar2 %.0f total %.0f" % tuple(pr[32:38] / st))
