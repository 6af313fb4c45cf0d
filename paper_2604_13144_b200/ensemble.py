"""Batched TE-PAI ensemble on the B200 engine (north_star items 1-4).

Host: the reference-identical sampler draws every circuit (``circuit_stream``
keyed by sample id, so the draw is independent of batching and rank count),
``packing`` turns it into gate words, and one ``tb_run_ensemble`` call runs the
persistent kernel over the whole batch.  Multi-GPU: one process per GPU, each
rank takes a contiguous range of sample ids, and the fixed-point (checkpoint,
site) sums are combined with a single ``all_reduce`` — the only collective of
the path.
"""

from __future__ import annotations

import ctypes
import math
import queue
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .estimator import FIX, aggregate_fixed
from .mps import SITE_VECTORS, TruncationPolicy
from .packing import TermTable, angle_table, pack_batch, pack_sampled, tepai_angles
from .pauli import Hamiltonian
from .rng import circuit_stream
from .sampling import PaiConfig, circuit_weight_norm, sample_circuit


# The estimator sums hold round(2^40 v) per sample with |v| <= 1 (+ rounding),
# so a (checkpoint, site) row overflows int64 after ~2^23 samples.  Every
# accumulation path checks its row counts against this bound.
MAX_SAMPLES_PER_ROW = int((2**63 - 1) // (FIX * (1.0 + 1e-6)))


def check_row_capacity(counts) -> None:
    """Raise before an int64 fixed-point row could wrap."""
    c = np.asarray(counts, dtype=np.int64)
    if c.size and int(c.max()) > MAX_SAMPLES_PER_ROW:
        raise OverflowError(f"{int(c.max())} samples in one estimator row exceed the 2^-40 fixed-point capacity "
                            f"({MAX_SAMPLES_PER_ROW}); flush the sums (aggregate and restart) before that")


def checkpoint_weights(ham: Hamiltonian, cfg: PaiConfig, checkpoints) -> np.ndarray:
    """||g||_1 of each prefix: circuit_weight_norm(H, PaiConfig(D, j, jT/N))
    (SURVEY.md §8(a) prefix semantics)."""
    return np.array([circuit_weight_norm(ham, PaiConfig(cfg.delta, int(j), j * cfg.total_time / cfg.n_steps, cfg.mode))
                     for j in checkpoints])


@dataclass
class PackedEnsemble:
    """Host-side input of one engine call."""

    n: int
    cap: int
    chi_cut: int
    floor: float
    words: np.ndarray
    offsets: np.ndarray
    ckpt_end: np.ndarray
    ckpt_sign: np.ndarray
    angle_cs: np.ndarray
    weights: np.ndarray
    obs_sites: np.ndarray
    init_vecs: np.ndarray
    sample_ids: np.ndarray
    nu: np.ndarray
    pi_local: bool = True
    init_mps: np.ndarray | None = None   # complex128 [n, cap, 2, cap] start state (hybrid fan-out)
    init_dims: np.ndarray | None = None  # int32 [n+1]
    init_center: int = 0

    @property
    def n_samples(self) -> int:
        return int(self.sample_ids.size)

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.words, self.offsets, self.ckpt_end, self.ckpt_sign, self.angle_cs,
                                      self.obs_sites, self.init_vecs))


def pack_ensemble(ham: Hamiltonian, cfg: PaiConfig, seed: int, sample_ids, labels, policy: TruncationPolicy,
                  checkpoints, obs_sites=None, pi_local: bool = True, init_state=None) -> PackedEnsemble:
    """Sample (reference-identical draws) and pack a batch of circuits.  With
    ``init_state`` (an ``MPSState``) every sample starts from that MPS instead
    of the product state ``labels`` (hybrid Trotter -> TE-PAI)."""
    n = ham.n
    if init_state is None and len(labels) != n:
        raise ValueError("initial-state labels do not match the chain length")
    hard = 2 ** (n // 2)
    cut = hard if policy.chi_cut is None else min(policy.chi_cut, hard)
    checkpoints = np.asarray(checkpoints, dtype=np.int64)
    if checkpoints.size and (np.any(np.diff(checkpoints) <= 0) or checkpoints[0] < 0 or checkpoints[-1] > cfg.n_steps):
        raise ValueError("checkpoints must be increasing step counts within [0, n_steps]")
    table = TermTable.of(ham)
    ids = np.asarray(list(sample_ids), dtype=np.int64)
    packed = []
    for sid in ids:
        circ = sample_circuit(ham, cfg, circuit_stream(seed, int(sid)), sample_id=int(sid))
        packed.append(pack_sampled(circ, table, checkpoints))
    words, offs, ce, cs = pack_batch(packed, int(checkpoints.size))
    obs = np.arange(n, dtype=np.int32) if obs_sites is None else np.asarray(obs_sites, dtype=np.int32)
    labs = labels if init_state is None else "0" * n
    init = np.stack([SITE_VECTORS[lab] for lab in labs]).astype(np.complex128)
    pe = PackedEnsemble(n, cut, cut, float(policy.svalue_floor), words, offs, ce, cs,
                        angle_table(tepai_angles(cfg.delta)), checkpoint_weights(ham, cfg, checkpoints), obs,
                        init.view(np.float64).reshape(n, 4).copy(), ids, np.diff(offs), pi_local)
    if init_state is not None:
        if init_state.n != n:
            raise ValueError(f"start state on {init_state.n} qubits, Hamiltonian has {n}")
        if init_state.max_bond() > cut:
            raise ValueError("start state bond dimension exceeds the truncation cap")
        st = init_state.copy()
        st.ensure_capacity(cut)
        if st.cap != cut:  # shrink a larger buffer to the ensemble capacity
            buf = np.zeros((n, cut, 2, cut), np.complex128)
            for q in range(n):
                buf[q, : st.dims[q], :, : st.dims[q + 1]] = st.buf[q, : st.dims[q], :, : st.dims[q + 1]]
            st.buf, st.cap = buf, cut
        pe.init_mps = np.ascontiguousarray(st.buf)
        pe.init_dims = st.dims.astype(np.int32)
        pe.init_center = int(st.center)
    return pe


@dataclass
class EnsembleRun:
    """Per-sample outputs and fixed-point sums of one (or several merged) calls."""

    n_samples: int
    values: np.ndarray | None     # [S, C, O] raw <Z_j>
    discarded: np.ndarray | None  # [S, C]
    ledger: np.ndarray | None     # [S, 4]
    sum_v: np.ndarray             # int64 [C, O]
    sum_v2: np.ndarray            # int64 [C, O]
    weights: np.ndarray           # [C]
    flops: float
    kernel_ms: float
    wall_s: float
    extra: dict = field(default_factory=dict)
    excluded: np.ndarray | None = None  # [S] first checkpoint left out of the sums (-1: none)
    counts: np.ndarray | None = None    # [C] samples summed into each checkpoint row
    states: np.ndarray | None = None    # complex128 [S, n, cap, 2, cap] final MPS per sample (retain_states)
    state_dims: np.ndarray | None = None  # int32 [S, n+1]
    state_center: np.ndarray | None = None  # int32 [S]
    sample_ms: np.ndarray | None = None  # [S] device time per sample (time_samples)
    sample_ids: np.ndarray | None = None
    nu: np.ndarray | None = None         # [S] gate-list length per sample
    signs: np.ndarray | None = None      # int8 [S, C] sign(g) of each prefix

    def row_counts(self) -> np.ndarray:
        """Samples that contributed to each checkpoint row of the sums."""
        if self.counts is not None:
            return self.counts
        return np.full(self.sum_v.shape[0], self.n_samples, dtype=np.int64)

    def stats(self) -> dict:
        return aggregate_fixed(self.sum_v, self.sum_v2, self.row_counts(), self.weights)


def excluded_counts(excluded: np.ndarray, n_ckpt: int) -> np.ndarray:
    """Per-checkpoint count of samples whose rows were left out (checkpoints
    from excluded[s] on; -1 = none)."""
    ex = np.asarray(excluded, dtype=np.int64)
    drop = np.zeros(n_ckpt, np.int64)
    for e in ex[ex >= 0]:
        drop[e:] += 1
    return drop


def run_packed(p: PackedEnsemble, device: int = 0, keep_values: bool = True, retain_states: bool = False,
               time_samples: bool = False) -> EnsembleRun:
    """One end-to-end engine call with host buffers (``tb_run_ensemble``).
    ``retain_states`` keeps every sample's final MPS (signed-mixture
    post-processing; memory n cap^2 per sample);
    ``time_samples`` records each sample's device time (cost report)."""
    S, C, O = p.n_samples, p.ckpt_end.shape[1] if p.ckpt_end.ndim == 2 else 0, p.obs_sites.size
    values = np.zeros((S, C, O)) if keep_values else None
    disc = np.zeros((S, C)) if keep_values else None
    ledger = np.zeros((S, 4))
    sv = np.zeros((C, O), np.int64)
    sv2 = np.zeros((C, O), np.int64)
    flops = np.zeros(1)
    kms = np.zeros(1, np.float32)
    excl = np.full(S, -1, np.int32)
    check_row_capacity([S])
    states = np.zeros((S, p.n, p.cap, 2, p.cap), np.complex128) if retain_states else None
    sdims = np.zeros((S, p.n + 1), np.int32) if retain_states else None
    scen = np.zeros(S, np.int32) if retain_states else None
    sms = np.zeros(S) if time_samples else None
    arrays = [np.ascontiguousarray(x) for x in (p.words, p.offsets, p.ckpt_end, p.ckpt_sign, p.angle_cs,
                                                 p.weights, p.obs_sites, p.init_vecs)]
    w, off, ce, cs, ang, wt, obs, iv = arrays
    desc = _lib.EnsembleDesc(p.n, p.cap, p.chi_cut, int(p.pi_local), p.floor, S, C, O, ang.shape[0],
                             w.ctypes.data, off.ctypes.data, ce.ctypes.data, cs.ctypes.data, ang.ctypes.data,
                             wt.ctypes.data, obs.ctypes.data, iv.ctypes.data,
                             p.init_mps.ctypes.data if p.init_mps is not None else None,
                             p.init_dims.ctypes.data if p.init_dims is not None else None, p.init_center, 0)
    out = _lib.EnsembleOut(values.ctypes.data if values is not None else None,
                           disc.ctypes.data if disc is not None else None, ledger.ctypes.data,
                           sv.ctypes.data, sv2.ctypes.data, flops.ctypes.data, kms.ctypes.data, excl.ctypes.data,
                           *(x.ctypes.data if x is not None else None for x in (states, sdims, scen, sms)))
    ctx = _lib.context(device)
    t0 = time.perf_counter()
    _lib.check(_lib.load().tb_run_ensemble(ctx, ctypes.byref(desc), ctypes.byref(out)), ctx)
    wall = time.perf_counter() - t0
    counts = S - excluded_counts(excl, C)
    return EnsembleRun(S, values, disc, ledger, sv, sv2, p.weights, float(flops[0]), float(kms[0]), wall,
                       excluded=excl, counts=counts, states=states, state_dims=sdims, state_center=scen,
                       sample_ms=sms, sample_ids=p.sample_ids, nu=p.nu, signs=p.ckpt_sign)


def run_ensemble(ham: Hamiltonian, cfg: PaiConfig, seed: int, sample_ids, init_labels, policy: TruncationPolicy,
                 checkpoints, observables=None, pi_local: bool = True, device: int = 0,
                 keep_values: bool = True, init_state=None, retain_states: bool = False,
                 time_samples: bool = False) -> EnsembleRun:
    """Batched ensemble: <Z_j> at each checkpoint step for every sample, plus the
    signed fixed-point sums of the estimator."""
    p = pack_ensemble(ham, cfg, seed, sample_ids, init_labels, policy, checkpoints, observables, pi_local,
                      init_state)
    return run_packed(p, device, keep_values, retain_states, time_samples)


def broadcast_state(state, src: int = 0, group=None):
    """Fan one MPS out to every rank (config 5): snapshot bytes (mps.py:296-338
    format) through one torch.distributed broadcast."""
    import torch
    import torch.distributed as dist

    from .mps import snapshot_from_bytes, snapshot_to_bytes

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    if dist.get_rank(group) == src:
        raw = np.frombuffer(snapshot_to_bytes(state), dtype=np.uint8)
        size = torch.tensor([raw.size], dtype=torch.int64, device=dev)
    else:
        size = torch.zeros(1, dtype=torch.int64, device=dev)
    dist.broadcast(size, src, group=group)
    buf = torch.from_numpy(raw.copy()).to(dev) if dist.get_rank(group) == src else torch.zeros(
        int(size[0]), dtype=torch.uint8, device=dev)
    dist.broadcast(buf, src, group=group)
    return state if dist.get_rank(group) == src else snapshot_from_bytes(buf.cpu().numpy().tobytes())


def run_hybrid(ham: Hamiltonian, trotter_steps: int, t0: float, cfg: PaiConfig, seed: int, sample_ids, init_labels,
               policy: TruncationPolicy, checkpoints, observables=None, pi_local: bool = True, device: int = 0,
               keep_values: bool = True, group=None):
    """Config 5: deterministic first-order Trotter evolution to t0 on the GPU
    (``run_circuit`` on the continuous-angle circuit, trotter.py:48-57), then a
    TE-PAI extension over ``cfg.total_time`` where every sample starts from that
    MPS.  Under torch.distributed rank 0 evolves and the
    snapshot is broadcast; each rank then runs its own ``sample_ids`` shard.
    Returns (EnsembleRun, start MPSState)."""
    from .mps import init_product_state, run_circuit
    from .trotter import build_trotter_circuit

    try:
        import torch.distributed as dist

        distributed = dist.is_available() and dist.is_initialized()
    except ImportError:
        distributed = False
    state = None
    if not distributed or dist.get_rank(group) == 0:
        state = init_product_state(init_labels)
        run_circuit(state, build_trotter_circuit(ham, t0, trotter_steps), policy)
    if distributed:
        state = broadcast_state(state, 0, group)
    run = run_ensemble(ham, cfg, seed, sample_ids, init_labels, policy, checkpoints, observables, pi_local, device,
                       keep_values, init_state=state)
    return run, state



def shard_range(n_samples: int, rank: int, world: int) -> range:
    """Contiguous sample-id range of one rank."""
    lo = (n_samples * rank) // world
    hi = (n_samples * (rank + 1)) // world
    return range(lo, hi)


def allreduce_sums(run: EnsembleRun, group=None) -> EnsembleRun:
    """Combine per-rank fixed-point sums with ONE all_reduce (int64, exact and
    order-independent).  Packs [sum_v, sum_v2, n_samples] in one tensor."""
    import torch
    import torch.distributed as dist

    C, O = run.sum_v.shape
    flat = np.concatenate([run.sum_v.ravel(), run.sum_v2.ravel(), run.row_counts().astype(np.int64),
                           np.array([run.n_samples], np.int64)])
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(flat).to(dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    t = t.cpu().numpy()
    counts = t[2 * C * O: 2 * C * O + C].copy()
    check_row_capacity(counts)
    return EnsembleRun(int(t[-1]), None, None, None, t[: C * O].reshape(C, O).copy(),
                       t[C * O: 2 * C * O].reshape(C, O).copy(), run.weights, run.flops, run.kernel_ms,
                       run.wall_s, dict(run.extra), counts=counts)


def slot_order(words: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Slot processing order for one step: decreasing predicted cost, so the
    persistent CTAs' atomic slot queue approximates longest-processing-time
    scheduling.  The cost of a segment is its number of two-site SVD updates:
    1 per adjacent two-site gate and 2 (b - a - 1) + 1 per non-adjacent (ring)
    gate, whose swap sweep costs one update per swap (_kernel.py:203-215)."""
    a = (words & 0xFF).astype(np.int64)
    b = ((words >> 8) & 0xFF).astype(np.int64)
    cost = np.where(b == 0xFF, 0, np.where(b - a > 1, 2 * (b - a - 1) + 1, 1))
    c = np.concatenate([[0], np.cumsum(cost)])
    offs = np.asarray(offsets, dtype=np.int64)
    seg = c[offs[1:]] - c[offs[:-1]]
    return np.argsort(-seg, kind="stable").astype(np.int32)


@dataclass
class StepPlan:
    """Host inputs of one pipeline step (one checkpoint segment per slot)."""

    words: np.ndarray      # uint32, all slots' segments concatenated
    offsets: np.ndarray    # int64 [S+1]
    ckpt_end: np.ndarray   # int32 [S, 1]
    ckpt_sign: np.ndarray  # int8 [S, 1]
    reset: np.ndarray      # uint8 [S]
    sum_row: np.ndarray    # int32 [S, 1]
    completes: int         # samples finished by this step
    order: np.ndarray | None = None  # int32 [S] slot processing order (decreasing predicted cost)
    slot_sample: np.ndarray | None = None  # int64 [S] sample id each slot advances this step

    def nbytes(self) -> int:
        """Host->device bytes of this step's inputs."""
        return sum(x.nbytes for x in (self.words, self.offsets, self.ckpt_end, self.ckpt_sign, self.reset,
                                      self.sum_row) + ((self.order,) if self.order is not None else ()))


class SlotPipeline:
    """Continuous batching of ensemble members over persistent GPU slots.

    Every slot keeps its MPS resident in HBM.  Each ``step`` advances every
    slot by one checkpoint segment of its current circuit (and measures
    <Z_j>); a slot that finished its circuit restarts from the product state
    with the next sample id.  Checkpoint c of every sample accumulates into
    estimator row c, so the statistics equal those of ``run_ensemble`` on the
    same ids.

    The pipeline owns a private engine context, so its slot pool is never
    aliased by another pipeline or by ``run_circuit`` / ``run_ensemble`` /
    ``tb_svd`` calls; the engine additionally refuses to continue a slot whose
    state belongs to an older workspace generation.  ``run`` overlaps the host
    producer (sampling + packing of step k+1, reference sampler
    sampling.py:244-321) with the engine call of step k.
    """

    def __init__(self, ham: Hamiltonian, cfg: PaiConfig, seed: int, labels, policy: TruncationPolicy,
                 checkpoints, n_slots: int | None = None, observables=None, pi_local: bool = True,
                 device: int = 0, first_sample: int = 0, sample_stride: int = 1, init_state=None,
                 step_engine=None):
        self.ham, self.cfg, self.seed, self.device = ham, cfg, seed, device
        self.labels, self.policy = labels, policy
        self.checkpoints = np.asarray(checkpoints, dtype=np.int64)
        if self.checkpoints[-1] != cfg.n_steps:
            raise ValueError("the last checkpoint must be the end of the circuit")
        self.proto = pack_ensemble(ham, cfg, seed, [], labels, policy, self.checkpoints, observables, pi_local,
                                   init_state)
        # ``step_engine`` replaces the device call of a step (host-logic tests on
        # machines without a GPU inject a CPU checker through it); the product
        # path always goes through the C ABI
        self.step_engine = step_engine
        if step_engine is None:
            self._own = _lib.PrivateContext(device)
            self.ctx = self._own.ctx
            sms = _lib.load().tb_num_ctas(self.ctx, int(self.proto.cap))  # persistent CTAs for this bond capacity
        else:
            if not n_slots:
                raise ValueError("an injected step engine needs an explicit n_slots")
            self._own, self.ctx, sms = None, None, int(n_slots)
        self.n_slots = int(n_slots or sms)  # > sms: slots queue onto the persistent CTAs
        self.table = TermTable.of(ham)
        self.next_id = first_sample
        self.stride = sample_stride
        self.slot_pack = [None] * self.n_slots
        self.slot_seg = [0] * self.n_slots
        self.slot_id = np.full(self.n_slots, -1, np.int64)
        C, O = self.checkpoints.size, self.proto.obs_sites.size
        self.sum_v = np.zeros((C, O), np.int64)
        self.sum_v2 = np.zeros((C, O), np.int64)
        self.row_count = np.zeros(C, np.int64)  # samples summed into each row (committed steps only)
        self.excluded: dict[int, int] = {}      # sample id -> first checkpoint left out (non-converged SVD)
        self.completed = 0
        self.flops = 0.0

    def close(self) -> None:
        """Release the private engine context (and its slot pool)."""
        if self._own is not None:
            self._own.close()

    def _new_sample(self):
        sid = self.next_id
        self.next_id += self.stride
        circ = sample_circuit(self.ham, self.cfg, circuit_stream(self.seed, sid), sample_id=sid)
        return sid, pack_sampled(circ, self.table, self.checkpoints)

    def plan(self) -> StepPlan:
        """Host-side packing of the next step (advances the host schedule)."""
        S, C = self.n_slots, self.checkpoints.size
        segs, reset = [], np.zeros(S, np.uint8)
        sign = np.zeros((S, 1), np.int8)
        row = np.zeros((S, 1), np.int32)
        ids = np.zeros(S, np.int64)
        completes = 0
        for b in range(S):
            if self.slot_pack[b] is None or self.slot_seg[b] == C:
                self.slot_id[b], self.slot_pack[b] = self._new_sample()
                self.slot_seg[b] = 0
                reset[b] = 1
            p, c = self.slot_pack[b], self.slot_seg[b]
            lo = 0 if c == 0 else int(p.ckpt_end[c - 1])
            segs.append(p.words[lo: int(p.ckpt_end[c])])
            sign[b, 0] = p.ckpt_sign[c]
            row[b, 0] = c
            ids[b] = self.slot_id[b]
            self.slot_seg[b] = c + 1
            completes += int(c + 1 == C)
        offs = np.zeros(S + 1, np.int64)
        offs[1:] = np.cumsum([s.size for s in segs])
        ends = np.diff(offs).astype(np.int32).reshape(S, 1)
        words = np.concatenate(segs).astype(np.uint32)
        return StepPlan(words, offs, ends, sign, reset, row, completes, slot_order(words, offs), ids)

    def planned(self, n_steps: int, depth: int = 2):
        """Yield the next ``n_steps`` plans, produced ahead by a background
        thread (the engine call releases the GIL, so sampling and packing of
        step k+1 overlap step k on the GPU)."""
        q: queue.Queue = queue.Queue(maxsize=max(1, depth))
        err: list = []

        def work():
            try:
                for _ in range(n_steps):
                    q.put(self.plan())
            except BaseException as e:  # noqa: BLE001 - re-raised in the consumer
                err.append(e)
                q.put(None)

        th = threading.Thread(target=work, name="tepai-producer", daemon=True)
        th.start()
        for _ in range(n_steps):
            p = q.get()
            if p is None:
                raise err[0]
            yield p
        th.join()

    def run(self, n_steps: int, overlap: bool = True, on_step=None) -> list[float]:
        """Advance the pipeline by ``n_steps`` steps through the host-buffer C
        ABI (``tb_step``); returns the per-step kernel times in ms."""
        plans = self.planned(n_steps) if overlap else (self.plan() for _ in range(n_steps))
        ms = []
        for i, p in enumerate(plans):
            ms.append(self.step_host(p))
            if on_step is not None:
                on_step(i, ms[-1])
        return ms

    def _desc(self, ptrs, S):
        p = self.proto
        base = _lib.EnsembleDesc(p.n, p.cap, p.chi_cut, int(p.pi_local), p.floor, S, 1, p.obs_sites.size,
                                 p.angle_cs.shape[0], ptrs["words"], ptrs["offsets"], ptrs["ckpt_end"],
                                 ptrs["ckpt_sign"], ptrs["angle_cs"], None, ptrs["obs"], ptrs["init"],
                                 ptrs.get("init_mps"), ptrs.get("init_dims"), p.init_center, 0)
        return _lib.StepDesc(base, ptrs["reset"], ptrs["sum_row"], ptrs.get("order"))

    def _commit(self, plan: StepPlan, excl: np.ndarray) -> None:
        """Row counts of a finished step: every slot whose checkpoint was
        summed; a slot flagged by the engine (non-converged SVD) is dropped and
        its sample remembered."""
        ok = excl < 0
        np.add.at(self.row_count, plan.sum_row[ok, 0], 1)
        for b in np.flatnonzero(~ok):
            sid = int(plan.slot_sample[b]) if plan.slot_sample is not None else -1
            self.excluded.setdefault(sid, int(plan.sum_row[b, 0]))
        self.completed += plan.completes

    def step_host(self, plan: StepPlan, values: np.ndarray | None = None, discarded: np.ndarray | None = None) -> float:
        """End-to-end step through ``tb_step`` with host buffers; returns kernel ms.
        ``values`` [S, 1, O] receives each slot's <Z_j>, ``discarded`` [S, 1]
        its circuit's cumulative discarded weight at this checkpoint."""
        S, O = self.n_slots, self.proto.obs_sites.size
        check_row_capacity(self.row_count + 1)
        if self.step_engine is not None:
            excl = np.full(S, -1, np.int32)
            vals = values if values is not None else np.zeros((S, 1, O))
            ms = float(self.step_engine(self, plan, vals, excl))
            self._commit(plan, excl)
            return ms
        keep = [plan.words, plan.offsets, plan.ckpt_end, plan.ckpt_sign, plan.reset, plan.sum_row,
                self.proto.angle_cs, self.proto.obs_sites, self.proto.init_vecs]
        keep = [np.ascontiguousarray(x) for x in keep]
        ptrs = dict(zip(["words", "offsets", "ckpt_end", "ckpt_sign", "reset", "sum_row", "angle_cs", "obs", "init"],
                        [x.ctypes.data for x in keep]))
        if plan.order is not None:
            keep.append(np.ascontiguousarray(plan.order, dtype=np.int32))
            ptrs["order"] = keep[-1].ctypes.data
        if self.proto.init_mps is not None:
            ptrs["init_mps"] = self.proto.init_mps.ctypes.data
            ptrs["init_dims"] = self.proto.init_dims.ctypes.data
        desc = self._desc(ptrs, S)
        vals = values if values is not None else np.zeros((S, 1, O))
        flops = np.zeros(1)
        kms = np.zeros(1, np.float32)
        excl = np.full(S, -1, np.int32)
        out = _lib.EnsembleOut(vals.ctypes.data, discarded.ctypes.data if discarded is not None else None, None,
                               self.sum_v.ctypes.data, self.sum_v2.ctypes.data, flops.ctypes.data, kms.ctypes.data,
                               excl.ctypes.data)
        _lib.check(_lib.load().tb_step(self.ctx, ctypes.byref(desc), ctypes.byref(out), self.sum_v.shape[0]), self.ctx)
        self.flops += float(flops[0])
        self._commit(plan, excl)
        return float(kms[0])

    def upload(self, plan: StepPlan, stream=None):
        """Device copies of a step's inputs (torch tensors on this device),
        copied asynchronously from pinned host memory on ``stream``."""
        import torch

        dev = torch.device("cuda", self.device)
        arrs = (("words", plan.words.view(np.int32)), ("offsets", plan.offsets), ("ckpt_end", plan.ckpt_end),
                ("ckpt_sign", plan.ckpt_sign), ("reset", plan.reset), ("sum_row", plan.sum_row))
        if plan.order is not None:
            arrs += (("order", np.asarray(plan.order, dtype=np.int32)),)
        t = {}
        with torch.cuda.stream(stream) if stream is not None else _nullctx():
            for k, v in arrs:
                h = torch.from_numpy(np.ascontiguousarray(v)).pin_memory()
                t[k] = h.to(dev, non_blocking=True)
                t["_pin_" + k] = h  # keep the pinned source alive until the copy ran
        t["plan"] = plan
        return t

    def device_state(self):
        """Device-resident constant inputs and outputs for ``step_device``."""
        import torch

        dev = torch.device("cuda", self.device)
        S, C, O = self.n_slots, self.checkpoints.size, self.proto.obs_sites.size
        return {
            "angle_cs": torch.from_numpy(self.proto.angle_cs).to(dev),
            "obs": torch.from_numpy(self.proto.obs_sites).to(dev),
            "init": torch.from_numpy(self.proto.init_vecs).to(dev),
            "values": torch.zeros((S, 1, O), dtype=torch.float64, device=dev),
            "sum_v": torch.from_numpy(self.sum_v).to(dev),
            "sum_v2": torch.from_numpy(self.sum_v2).to(dev),
            "flops": torch.zeros(1, dtype=torch.float64, device=dev),
            "excl": torch.full((S,), -1, dtype=torch.int32, device=dev),
            "rows_ok": torch.zeros(C, dtype=torch.int64, device=dev),
            "rows_bad": torch.zeros(C, dtype=torch.int64, device=dev),
            **({"init_mps": torch.from_numpy(self.proto.init_mps.view(np.float64)).to(dev),
                "init_dims": torch.from_numpy(self.proto.init_dims).to(dev)} if self.proto.init_mps is not None else {}),
        }

    def step_device(self, t: dict, ds: dict, stream_ptr: int) -> None:
        """Device-resident step through ``tb_step_device`` on ``stream_ptr``
        (asynchronous; ``sync_from_device`` brings sums, counts and status back)."""
        import torch

        S = self.n_slots
        ptrs = {k: t[k].data_ptr() for k in ("words", "offsets", "ckpt_end", "ckpt_sign", "reset", "sum_row")}
        if "order" in t:
            ptrs["order"] = t["order"].data_ptr()
        ptrs.update(angle_cs=ds["angle_cs"].data_ptr(), obs=ds["obs"].data_ptr(), init=ds["init"].data_ptr())
        if "init_mps" in ds:
            ptrs.update(init_mps=ds["init_mps"].data_ptr(), init_dims=ds["init_dims"].data_ptr())
        desc = self._desc(ptrs, S)
        stream = torch.cuda.ExternalStream(stream_ptr) if stream_ptr else torch.cuda.current_stream()
        with torch.cuda.stream(stream):
            ds["excl"].fill_(-1)
        out = _lib.EnsembleOut(ds["values"].data_ptr(), None, None, ds["sum_v"].data_ptr(), ds["sum_v2"].data_ptr(),
                               ds["flops"].data_ptr(), None, ds["excl"].data_ptr())
        _lib.check(_lib.load().tb_step_device(self.ctx, ctypes.byref(desc), ctypes.byref(out), stream_ptr), self.ctx)
        with torch.cuda.stream(stream):
            rows = t["sum_row"][:, 0].long()
            bad = (ds["excl"] >= 0).long()
            ds["rows_ok"].index_add_(0, rows, 1 - bad)
            ds["rows_bad"].index_add_(0, rows, bad)
        self.completed += t["plan"].completes

    def sync_from_device(self, ds: dict) -> None:
        """Copy the device-resident sums, row counts and FLOPs of ``step_device``
        calls back into this pipeline (after which ``stats`` is current), and
        surface the engine's sticky status (non-convergence is reported per
        row through ``rows_bad``; a stale-slot continuation raises)."""
        import torch

        torch.cuda.synchronize(self.device)
        self.sum_v[...] = ds["sum_v"].cpu().numpy()
        self.sum_v2[...] = ds["sum_v2"].cpu().numpy()
        self.row_count += ds["rows_ok"].cpu().numpy()
        bad = ds["rows_bad"].cpu().numpy()
        if bad.any():
            self.excluded.setdefault(-1, int(np.flatnonzero(bad)[0]))
        ds["rows_ok"].zero_()
        ds["rows_bad"].zero_()
        self.flops += float(ds["flops"].item())
        ds["flops"].zero_()
        st = _lib.take_status(self.ctx)
        if st & 4:
            raise ValueError("a slot was continued after its workspace generation changed; reset every slot")

    def stats(self) -> dict:
        """Estimator over the samples summed into each checkpoint row."""
        out = {}
        for c in range(self.checkpoints.size):
            n = int(self.row_count[c])
            if n:
                st = aggregate_fixed(self.sum_v[c:c + 1], self.sum_v2[c:c + 1], n, self.proto.weights[c:c + 1])
                out[c] = {k: v[0] for k, v in st.items()}
        return out


def pipeline_shard(ham: Hamiltonian, cfg: PaiConfig, seed: int, labels, policy: TruncationPolicy, checkpoints,
                   n_slots: int | None = None, rank: int = 0, world: int = 1, **kw) -> SlotPipeline:
    """Rank ``rank``'s pipeline of a ``world``-rank job: it draws sample ids
    rank, rank + world, rank + 2 world, ... (the draw of id i
    is ``circuit_stream(seed, i)`` on every rank, so the union over ranks is
    the 1-rank id set and the reduced sums are bit-identical to it)."""
    return SlotPipeline(ham, cfg, seed, labels, policy, checkpoints, n_slots=n_slots, first_sample=rank,
                        sample_stride=world, **kw)


def reduce_pipeline(pipe: SlotPipeline, group=None) -> EnsembleRun:
    """The path's only collective: ONE all_reduce of the pipeline's int64
    fixed-point sums, per-row counts and completed-sample count over the
    process group (NCCL on GPUs, gloo on CPU).  Identity at world 1."""
    run = EnsembleRun(pipe.completed, None, None, None, pipe.sum_v.copy(), pipe.sum_v2.copy(), pipe.proto.weights,
                      pipe.flops, 0.0, 0.0, counts=pipe.row_count.copy())
    try:
        import torch.distributed as dist

        distributed = dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1
    except ImportError:
        distributed = False
    return allreduce_sums(run, group) if distributed else run


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
