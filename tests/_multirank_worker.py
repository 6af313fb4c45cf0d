"""Worker for the multi-rank determinism tests (launched by
``torch.distributed.run``; see tests/test_multirank.py).  Runs the C1-size
slot pipeline shard of this rank — ids rank, rank+world, ... — for a fixed
number of full circuit lifecycles, reduces with ``reduce_pipeline`` (one
all_reduce over gloo) and rank 0 writes the sums.

  --engine oracle : the CPU checker stands in for the device call (no GPU)
  --engine gpu    : the real engine through the C ABI (one private context
                    per rank; all ranks may share one GPU: their kernels are
                    independent and only the final gloo all_reduce joins them)
"""

import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2604_13144_b200 as tb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--engine", choices=["oracle", "gpu"], required=True)
    ap.add_argument("--slots", type=int, required=True, help="total slots over all ranks")
    ap.add_argument("--lifecycles", type=int, default=2)
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    ham = tb.build_spin_ring(8, 1.0, 0)
    cfg = tb.PaiConfig(math.pi / 2**7, 100, 1.0)
    ck = np.arange(10, 101, 10)
    eng = None
    if a.engine == "oracle":
        from oracle_slot_engine import OracleSlotEngine

        eng = OracleSlotEngine()
    else:
        import __graft_entry__

        __graft_entry__.build()
    pipe = tb.pipeline_shard(ham, cfg, 1, "01" * 4, tb.TruncationPolicy(16), ck, n_slots=a.slots // world, rank=rank,
                             world=world, step_engine=eng)
    pipe.run(a.lifecycles * ck.size)
    run = tb.reduce_pipeline(pipe)
    if rank == 0:
        np.savez(a.out, sum_v=run.sum_v, sum_v2=run.sum_v2, counts=run.row_counts(), n=run.n_samples)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
