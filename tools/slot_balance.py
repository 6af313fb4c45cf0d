"""Load balance of the slot-mode step (bench definition): per launch, kernel
time vs the mean per-CTA busy time (clock64 counter prof[7] / CTAs / clock).
usage: python tools/slot_balance.py [steps] [slots]"""
import os, sys; sys.path.insert(0, "."); import __graft_entry__  # noqa: E702
# the library path is bound when the package is first imported (inside build()): set it before
os.environ.setdefault("TB_PROFILE", "1"); os.environ.setdefault("TB_LIB", __graft_entry__.LIB_PROF)  # phase counters: diagnostics build
__graft_entry__.build(profile=True)
import math, sys
import numpy as np
sys.path.insert(0, ".")
import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import _lib
from paper_2604_13144_b200.ensemble import SlotPipeline

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
slots = int(sys.argv[2]) if len(sys.argv) > 2 else None
ham = tb.build_spin_ring(32, 1.0, 4)
cfg = tb.PaiConfig(math.pi / 2**7, 200, 2.0)
pipe = SlotPipeline(ham, cfg, 5, "01" * 16, tb.TruncationPolicy(64, 1e-12), np.arange(10, 201, 10), n_slots=slots)
ctas = min(pipe.n_slots, 148)
prev = _lib.debug_profile(ctx=pipe.ctx).astype(np.float64)
for i in range(steps):
    ms = pipe.step_host(pipe.plan())
    pr = _lib.debug_profile(ctx=pipe.ctx).astype(np.float64)
    busy = pr[7] / ctas / 1.965e6  # the counters are reset per launch
    prev = pr
    print(f"step {i}: slots {pipe.n_slots} kernel {ms:.0f} ms, mean CTA busy {busy:.0f} ms, balance {busy / ms:.3f}")
