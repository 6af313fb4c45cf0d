"""Benchmark: TE-PAI circuit samples/sec on config 3 (N=32 disordered
Heisenberg ring, chi=64, complex128) and the % of the FP64 roofline.

A *step* is one pass of the hot path over one batch: every in-flight circuit
(S slots, by default two per SM = 296 on a B200, queued onto one persistent
CTA per SM in decreasing order of predicted cost) advances by one checkpoint
segment (10 of its 200 Trotter steps) and its <Z_j> are measured and added to
the signed estimator sums; a slot whose circuit finished restarts with the
next sample id (continuous batching).  20 steps = one full circuit per slot,
so samples/s = slots * K / 20 / T (sample-equivalents).  All slots start at
step 0; the default window (W=3, K=20, as the driver's W=5, K=20) times
exactly one full lifecycle per slot — every segment index 0..19 once,
segments 3..19 of the first circuits and 0..2 of the next.

``value`` uses the device time of the K persistent-kernel launches (inputs
already in HBM when each launch starts); ``e2e`` is the wall time of the same
K steps through the host-buffer C ABI call ``tb_step``: the host producer
thread (reference-identical sampler + packing, running ahead of the engine),
H2D of the step's gate words, the kernel, D2H of <Z_j>, the sums and the
per-slot exclusion flags, and the final reduction of the estimator sums.

``cpu_baseline`` (rank 0, N=1) times the numpy port of the reference engine
(oracle/, pinned bit-identical to the un-jitted reference) on every host core:
one circuit per core through one full 20-segment lifecycle, free-running.

``--impl reference`` is the reference arm: the same port on every host core
over the same W + K segment window, timed free-running (last end - first
start, no per-step barriers), plus — when the unmodified reference is
installed under baseline/_ref — that package itself (NUMBA_DISABLE_JIT=1)
over the first half of the lifecycle as a second CPU figure.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

# one BLAS thread per process: the CPU arm forks one worker per core, and a
# multithreaded BLAS inherited across fork would oversubscribe the host
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TE-PAI circuit samples/sec (N=32, χ=64, complex128) and % of FP64 roofline"
UNIT = "samples/s"
FP64_PEAK_TFLOPS = 37.08  # measured DMMA rate on this pool's B200 (profiles/r01_fp64_peak.txt)
C3 = dict(n=32, chi=64, ham_seed=4, circ_seed=5, n_steps=200, total_time=2.0, every=10)
WORKLOAD = ("C3: N=32 periodic disordered Heisenberg ring (h_j~U[-1,1], seed 4), Neel state, T=2.0 in 200 "
            "Trotter steps, Delta=pi/2^7, circuits from seed 5, chi_max=64, floor 1e-12, <Z_j> all j at 20 checkpoints")


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self._stop = index, [], threading.Event()
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > i + 2 and r[i + 2] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def c3_objects():
    import paper_2604_13144_b200 as tb

    ham = tb.build_spin_ring(C3["n"], 1.0, C3["ham_seed"])
    cfg = tb.PaiConfig(math.pi / 2**7, C3["n_steps"], C3["total_time"])
    pol = tb.TruncationPolicy(chi_cut=C3["chi"], svalue_floor=1e-12)
    ck = np.arange(C3["every"], C3["n_steps"] + 1, C3["every"])
    return tb, ham, cfg, pol, ck


# ---------------------------------------------------------------------------
# CPU arm: the reference engine's CPU path, one process per host core
# ---------------------------------------------------------------------------
REF_SITE = os.path.join(ROOT, "baseline", "_ref")  # unmodified reference (pip --target, git-ignored)


def _cpu_worker(args):
    """Advance circuit `sid` by n_segments checkpoint segments (restarting at
    each lifecycle end) and return the monotonic (start, end) of every segment.
    engine "port": the numpy restatement in oracle/ (pinned bit-identical to
    the un-jitted reference); "reference": the unmodified reference package
    from baseline/_ref with NUMBA_DISABLE_JIT=1 (its numba kernel does not
    compile under numba 0.65)."""
    sid, n_segments, engine = args
    from threadpoolctl import threadpool_limits

    threadpool_limits(1)
    tb, ham, cfg, pol, ck = c3_objects()
    circ = tb.sample_circuit(ham, cfg, tb.circuit_stream(C3["circ_seed"], sid), sample_id=sid)
    labels = "01" * (C3["n"] // 2)
    if engine == "reference":
        os.environ["NUMBA_DISABLE_JIT"] = "1"
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
        sys.path.insert(0, REF_SITE)
        import dataclasses

        import tepai

        zs = [tepai.PauliString.single(C3["n"], q, "Z") for q in range(C3["n"])]
        rc = tepai.sample_circuit(tepai.build_spin_ring(C3["n"], 1.0, C3["ham_seed"]),
                                  tepai.PaiConfig(math.pi / 2**7, C3["n_steps"], C3["total_time"]),
                                  tepai.rng.circuit_stream(C3["circ_seed"], sid), sample_id=sid)
        policy = tepai.TruncationPolicy(chi_cut=C3["chi"], svalue_floor=1e-12)

        def fresh():
            return tepai.init_product_state(labels)

        def advance(st, lo, hi):
            seg = dataclasses.replace(rc, term_index=rc.term_index[lo:hi], step_index=rc.step_index[lo:hi],
                                      kinds=rc.kinds[lo:hi], signs=rc.signs[lo:hi])
            tepai.run_circuit(st, seg, policy)
            return [tepai.expectation(st, z) for z in zs]
    else:
        from oracle.mps_oracle import OracleMPS

        def fresh():
            return OracleMPS(labels)

        def advance(st, lo, hi):
            st.run(circ.slice_entries(lo, hi).operations(), C3["chi"], 1e-12)
            return [st.expect({j: "Z"}) for j in range(C3["n"])]
    st, lo, stamps = None, 0, []
    for c in range(n_segments):
        if c % ck.size == 0:
            st, lo = fresh(), 0
        hi = int(np.searchsorted(circ.step_index, ck[c % ck.size]))
        t0 = time.monotonic()
        advance(st, lo, hi)
        stamps.append((t0, time.monotonic()))
        lo = hi
    return stamps


def cpu_run(n_segments: int, cores: int, engine: str = "port"):
    """`cores` free-running processes, each advancing its own circuit (ids
    0..cores-1) by n_segments segments; returns stamps[core][segment] =
    (start, end) on the shared monotonic clock."""
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        return np.array(pool.map(_cpu_worker, [(i, n_segments, engine) for i in range(cores)]))


def cpu_rate(stamps: np.ndarray, first: int, count: int):
    """Free-running throughput over segments [first, first + count): every
    core's work in that window / (last end - first start), no per-step
    barriers.  Returns (samples/s, wall seconds)."""
    wall = float(stamps[:, first + count - 1, 1].max() - stamps[:, first, 0].min())
    return stamps.shape[0] * count / 20.0 / wall, wall


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    cores = host_cores()
    steps = args.warmup + args.steps
    stamps = cpu_run(steps, cores, "port")
    value, wall = cpu_rate(stamps, args.warmup, args.steps)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (reference sampler, seeded)",
        "config": {"workload": WORKLOAD, "step": "one checkpoint segment (10 Trotter steps) per in-flight circuit",
                   "slots": cores, "parallelism": f"{cores} CPU processes"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"{cores} free-running processes, circuits 0..{cores - 1}, segments {args.warmup}.."
                                   f"{steps - 1} of the lifecycle timed (numpy port of the reference engine, zgesdd "
                                   f"via numpy LAPACK, 1 thread per process); wall = last end - first start"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_unmodified and os.path.isdir(os.path.join(REF_SITE, "tepai")):
        # second CPU figure: the unmodified reference itself, un-jitted, on the
        # same cores over the first half of the lifecycle, next to the port on
        # the same window (the port's arithmetic is the reference's)
        seg = args.unmodified_segments
        ref = cpu_run(seg, cores, "reference")
        rv, rw = cpu_rate(ref, 0, seg)
        pv, pw = cpu_rate(stamps, 0, min(seg, steps))
        line["reference_unmodified"] = {
            "value": rv, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(), "wall_s": rw,
            "sample": f"{cores} circuits x segments 0..{seg - 1} (bond-growth half of the lifecycle), unmodified "
                      "reference package (baseline/_ref, NUMBA_DISABLE_JIT=1)",
            "port_same_window": pv}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def run_b200(args):
    import torch

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__

    __graft_entry__.build()
    from paper_2604_13144_b200 import _lib
    from paper_2604_13144_b200.ensemble import pipeline_shard, reduce_pipeline

    tb, ham, cfg, pol, ck = c3_objects()
    # two slots per SM: the persistent CTAs take slots from a queue ordered by
    # predicted segment cost, which balances the per-segment work (0.87 -> 0.985
    # of the kernel time busy, tools/slot_balance.py)
    sms = _lib.load().tb_num_sms(_lib.context(local))
    pipe = pipeline_shard(ham, cfg, C3["circ_seed"], "01" * (C3["n"] // 2), pol, ck, n_slots=args.slots or 2 * sms,
                          rank=rank, world=world, device=local)
    S = pipe.n_slots
    # the host producer (reference sampler + packing) runs ahead in a thread for
    # every step, warm-up and timed alike: its work overlaps the engine calls,
    # and whatever it does not hide lands inside the e2e wall time
    plans = pipe.planned(args.warmup + args.steps)
    for i in range(args.warmup):
        ms = pipe.step_host(next(plans))
        print(f"[bench] warmup step {i}: {ms:.0f} ms", file=sys.stderr, flush=True)
    d2h = S * C3["n"] * 8 + 2 * pipe.sum_v.nbytes + S * 4
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kernel_ms, h2d, flops0 = [], [], pipe.flops
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(args.steps):
            p = next(plans)
            h2d.append(p.nbytes())
            kernel_ms.append(pipe.step_host(p))
            print(f"[bench] step {i}: {kernel_ms[-1]:.0f} ms", file=sys.stderr, flush=True)
        torch.cuda.synchronize()
        run = reduce_pipeline(pipe)  # the path's only collective: the estimator sums
        wall = time.perf_counter() - t0
    dev_s = sum(kernel_ms) / 1e3
    flops = pipe.flops - flops0
    if world > 1:
        t = torch.tensor([dev_s, wall], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, wall = float(t[0]), float(t[1])
        f = torch.tensor([flops], dtype=torch.float64, device="cuda")
        dist.all_reduce(f)
        flops = float(f[0])
    samples = world * S * args.steps / 20.0
    value = samples / dev_s
    e2e = samples / wall
    achieved = flops / dev_s / 1e12 / world  # per GPU, dominant kernel = the persistent ensemble kernel
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dev_s / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c128", "data": "synthetic (reference-identical seeded sampler, random disorder seed 4)",
        "config": {"workload": WORKLOAD, "slots_per_gpu": S, "ctas_per_gpu": min(S, sms),
                   "step": "one checkpoint segment (10 Trotter steps) of every in-flight circuit",
                   "samples_per_step": S / 20.0, "l2": "resident MPS state %.0f MB per GPU > 126 MB L2" % (
                       S * C3["n"] * 64 * 2 * 64 * 16 / 1e6),
                   "parallelism": f"dp{world} (sample sharding, one all_reduce of the estimator sums)",
                   "samples_completed": int(run.n_samples)},
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "peak_source": "measured FP64 DMMA rate (MEASURED_PEAKS.json has no FP64 entry)",
                     "flops": "SURVEY.md §8(d) algorithmic count (two-site contraction + LAPACK-nominal SVD + QR moves)"},
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": int(np.mean(h2d)), "d2h_bytes_per_step": int(d2h),
                "includes": "host sampling + packing (producer thread), H2D, kernel, D2H, final all_reduce"},
        "gpu_launches": 2 * args.steps,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        stamps = cpu_run(20, cores, "port")
        cpu, cwall = cpu_rate(stamps, 0, 20)
        line["cpu_baseline"] = {"value": cpu, "unit": UNIT, "cores": cores, "kind": "port", "cpu_model": cpu_model(),
                                "sample": f"{cores} circuits x one full 20-segment lifecycle, free-running processes "
                                          f"({cwall:.0f} s wall; numpy port of the reference engine, 1 thread each)"}
    pipe.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--slots", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-unmodified", action="store_true", help="reference arm: skip the unmodified-reference figure")
    ap.add_argument("--unmodified-segments", type=int, default=10)
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
