"""TEST INFRASTRUCTURE: a CPU stand-in for one ``tb_step`` launch, built on the
numpy oracle (``oracle/mps_oracle.py``).  Injected into ``SlotPipeline`` as
``step_engine`` so the pipeline's host logic — scheduling, continuous
batching, row accounting, sharding and the all_reduce — runs on machines
without a GPU.  It decodes the plan's gate words back into the reference's
lowered stream (mps.py:194-236 layout) and advances per-slot oracle states,
then adds the 2^-40 fixed-point values exactly as the kernel does
(record_checkpoint in csrc/tepai_b200.cu)."""

from __future__ import annotations

import math

import numpy as np

from oracle.mps_oracle import OracleMPS
from paper_2604_13144_b200.estimator import quantize


class OracleSlotEngine:
    def __init__(self):
        self.states: dict[int, OracleMPS] = {}

    def __call__(self, pipe, plan, vals, excl) -> float:
        angles = np.array([pipe.cfg.delta, -pipe.cfg.delta, math.pi])
        cut = pipe.proto.chi_cut
        for b in range(pipe.n_slots):
            if plan.reset[b] or b not in self.states:
                self.states[b] = OracleMPS(pipe.labels)
            st = self.states[b]
            w = plan.words[plan.offsets[b]: plan.offsets[b + 1]].astype(np.int64)
            if w.size:
                ga = w & 0xFF
                gbr = (w >> 8) & 0xFF
                gb = np.where(gbr == 0xFF, -1, gbr)
                pa, pb = (w >> 16) & 3, (w >> 18) & 3
                mr = (w >> 20) & 1
                ang = angles[w >> 22]
                nxt = np.where(mr == 1, ga + 1, ga)
                st.grow(cut)
                counters = np.zeros(4)
                st.run_lowered((ga, gb, pa, pb, ang, nxt), cut, pipe.proto.floor, counters,
                               bool(pipe.proto.pi_local))
            z = np.array([st.expect({int(j): "Z"}) for j in pipe.proto.obs_sites])
            vals[b, 0] = z
            row = int(plan.sum_row[b, 0])
            pipe.sum_v[row] += quantize(plan.ckpt_sign[b, 0] * z)
            pipe.sum_v2[row] += quantize(z * z)
        return 0.0
