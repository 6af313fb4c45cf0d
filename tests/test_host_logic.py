"""Host-side logic of the ensemble path (no GPU): slot scheduling cost,
fixed-point row capacity, per-row counts after engine exclusions, and the
overlapped producer of ``SlotPipeline`` (the device call replaced by the
oracle checker, tests/oracle_slot_engine.py)."""

import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import ensemble
from paper_2604_13144_b200.estimator import aggregate_fixed, quantize
from paper_2604_13144_b200.packing import encode
from oracle.mps_oracle import run_sample_checkpoints
from oracle_slot_engine import OracleSlotEngine


def _ring_word(a, b):
    return encode(np.array([a]), np.array([b]), np.array([1]), np.array([1]), np.array([0]), np.array([False]),
                  np.array([0]))


def test_slot_order_counts_segments_exactly_with_empty_tail():
    # offsets [0,1,3,3] with ring gates; the old reduceat clamp gave 9 instead of 18
    w = np.concatenate([_ring_word(0, 5), _ring_word(0, 5), _ring_word(0, 5)]).astype(np.uint32)
    offs = np.array([0, 1, 3, 3])
    per = 2 * (5 - 0 - 1) + 1
    order = ensemble.slot_order(w, offs)
    assert list(order) == [1, 0, 2]
    c = np.concatenate([[0], np.cumsum(np.full(3, per))])
    assert (c[offs[1:]] - c[offs[:-1]]).tolist() == [per, 2 * per, 0]
    assert list(ensemble.slot_order(np.zeros(0, np.uint32), np.zeros(4, np.int64))) == [0, 1, 2]


def test_row_capacity_guard():
    ensemble.check_row_capacity([ensemble.MAX_SAMPLES_PER_ROW])
    with pytest.raises(OverflowError):
        ensemble.check_row_capacity([1, ensemble.MAX_SAMPLES_PER_ROW + 1])
    # the bound really is where int64 would wrap
    q1 = int(quantize(1.0))
    assert ensemble.MAX_SAMPLES_PER_ROW * q1 < 2**63
    assert (ensemble.MAX_SAMPLES_PER_ROW + 10**5) * q1 > 2**63 * (1 - 1e-2)


def test_per_row_counts_after_exclusion():
    ex = np.array([-1, 2, -1, 0])
    np.testing.assert_array_equal(ensemble.excluded_counts(ex, 4), [1, 1, 2, 2])
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, size=(4, 4, 2))
    sv = np.zeros((4, 2), np.int64)
    sv2 = np.zeros((4, 2), np.int64)
    for s in range(4):
        for c in range(4):
            if ex[s] < 0 or c < ex[s]:
                sv[c] += quantize(v[s, c])
                sv2[c] += quantize(v[s, c] ** 2)
    counts = 4 - ensemble.excluded_counts(ex, 4)
    st = aggregate_fixed(sv, sv2, counts, np.ones(4))
    for c in range(4):
        rows = [s for s in range(4) if ex[s] < 0 or c < ex[s]]
        np.testing.assert_allclose(st["estimate"][c], v[rows, c].mean(axis=0), atol=1e-12)
        np.testing.assert_allclose(st["var_v"][c], v[rows, c].var(axis=0, ddof=1), atol=1e-10)


def _pipe(slots, eng, **kw):
    ham = tb.build_spin_ring(6, 1.0, 3)
    cfg = tb.PaiConfig(math.pi / 2**5, 30, 1.0)
    return ham, cfg, tb.SlotPipeline(ham, cfg, 7, "010101", tb.TruncationPolicy(8), [10, 20, 30], n_slots=slots,
                                     step_engine=eng, **kw)


def test_pipeline_producer_overlap_matches_serial_and_oracle():
    _, _, serial = _pipe(3, OracleSlotEngine())
    serial.run(6, overlap=False)
    ham, cfg, over = _pipe(3, OracleSlotEngine())
    seen = []
    over.run(6, overlap=True, on_step=lambda i, ms: seen.append(i))
    assert seen == list(range(6))
    np.testing.assert_array_equal(over.sum_v, serial.sum_v)
    np.testing.assert_array_equal(over.sum_v2, serial.sum_v2)
    np.testing.assert_array_equal(over.row_count, [6, 6, 6])
    assert over.completed == 6
    # the six samples 0..5, run whole by the oracle, give the same sums
    ref = np.zeros_like(over.sum_v)
    for i in range(6):
        circ = tb.sample_circuit(ham, cfg, tb.circuit_stream(7, i), sample_id=i)
        vals, signs, _, _ = run_sample_checkpoints(circ, "010101", 8, 1e-12, [10, 20, 30], pi_local=True)
        ref += quantize(signs[:, None] * vals)
    np.testing.assert_array_equal(over.sum_v, ref)
    st = over.stats()
    assert set(st) == {0, 1, 2}


def test_pipeline_engine_exclusion_drops_rows():
    base = OracleSlotEngine()

    def flaky(pipe, plan, vals, excl):
        ms = base(pipe, plan, vals, excl)
        # pretend slot 1's SVD failed in this step: the engine leaves its row out
        if plan.sum_row[1, 0] == 1:
            row = int(plan.sum_row[1, 0])
            z = vals[1, 0]
            pipe.sum_v[row] -= quantize(plan.ckpt_sign[1, 0] * z)
            pipe.sum_v2[row] -= quantize(z * z)
            excl[1] = 0
        return ms

    _, _, p = _pipe(2, flaky)
    p.run(3)
    np.testing.assert_array_equal(p.row_count, [2, 1, 2])
    assert p.excluded == {1: 1}


def test_producer_error_propagates():
    _, _, p = _pipe(2, OracleSlotEngine())

    def boom():
        raise RuntimeError("sampler failed")

    p.plan = boom
    with pytest.raises(RuntimeError, match="sampler failed"):
        p.run(2)
