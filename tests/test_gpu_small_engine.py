"""Small-problem engine (namespace tbs: bond capacity <= 32, two resident CTAs
per SM) against the full engine (TB_SMALL_ENGINE=0).  Both run the same
algorithm in the same order, so per-sample values, discarded weights and
ledgers agree to rounding (and each engine is bitwise reproducible run to
run); the C1 / C2 / TFIM parity tests
of test_gpu_parity.py run through the small engine by default and pin it to
the reference."""

import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import _lib, ensemble

pytestmark = pytest.mark.gpu


def test_cta_count_per_capacity(engine):
    lib, ctx = engine.load(), engine.context(0)
    sms = lib.tb_num_sms(ctx)
    assert lib.tb_num_ctas(ctx, 16) == 2 * sms
    assert lib.tb_num_ctas(ctx, 32) == 2 * sms
    assert lib.tb_num_ctas(ctx, 33) == sms
    assert lib.tb_num_ctas(ctx, 64) == sms


@pytest.mark.parametrize("n,chi,steps,ham_seed", [(8, 16, 40, 0), (12, 32, 40, 2), (10, 8, 30, 5)])
def test_small_engine_bit_identical_to_full_engine(engine, monkeypatch, n, chi, steps, ham_seed):
    ham = tb.build_spin_ring(n, 1.0, ham_seed)
    cfg = tb.PaiConfig(math.pi / 2**4, steps, 1.0)
    ck = np.arange(10, steps + 1, 10)
    sms = engine.load().tb_num_sms(engine.context(0))
    p = ensemble.pack_ensemble(ham, cfg, 3, range(2 * sms + 40), "01" * (n // 2), tb.TruncationPolicy(chi, 1e-12), ck)
    runs = {}
    for small in ("0", "1"):
        monkeypatch.setenv("TB_SMALL_ENGINE", small)
        runs[small] = ensemble.run_packed(p)
    a, b = runs["0"], runs["1"]
    # same algorithm and operation order; the two instantiations are separate
    # compilations (64 vs 128 registers per thread), so ptxas may fuse a
    # multiply-add differently here and there: agreement to rounding, not bitwise
    np.testing.assert_allclose(a.values, b.values, rtol=0, atol=1e-11)
    np.testing.assert_allclose(a.discarded, b.discarded, rtol=1e-6, atol=1e-15)
    np.testing.assert_array_equal(a.ledger[:, 0], b.ledger[:, 0])
    np.testing.assert_array_equal(a.ledger[:, 2], b.ledger[:, 2])
    assert np.abs(a.sum_v - b.sum_v).max() <= 2.0**40 * 1e-11 * p.n_samples
    assert a.flops == pytest.approx(b.flops, rel=1e-9)
    # each engine is bitwise reproducible run to run
    again = ensemble.run_packed(p)
    np.testing.assert_array_equal(again.values, b.values)
    np.testing.assert_array_equal(again.sum_v, b.sum_v)


def test_small_engine_slot_pipeline_default_slots(engine):
    """SlotPipeline sizes its default slot pool by tb_num_ctas: two slots per
    SM at chi <= 32; one lifecycle completes every slot's circuit."""
    n = 8
    ham = tb.build_spin_ring(n, 1.0, 0)
    cfg = tb.PaiConfig(math.pi / 2**7, 20, 0.2)
    ck = np.array([10, 20])
    pipe = tb.SlotPipeline(ham, cfg, 1, "01" * 4, tb.TruncationPolicy(16, 1e-12), ck)
    sms = _lib.load().tb_num_sms(pipe.ctx)
    assert pipe.n_slots == 2 * sms
    for p in pipe.planned(ck.size):
        pipe.step_host(p)
    assert pipe.completed == pipe.n_slots and not pipe.excluded
    pipe.close()
