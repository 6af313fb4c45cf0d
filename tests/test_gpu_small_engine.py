"""Small-problem engine (namespace tbs: bond capacity <= 32, two resident CTAs
per SM) against the full engine (TB_SMALL_ENGINE=0).  Both run the same
arithmetic in the same order, so per-sample values, discarded weights, ledgers
and the fixed-point sums must be bit-identical; the C1 / C2 / TFIM parity tests
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
    cfg = tb.PaiConfig(math.pi / 2**6, steps, 1.0)
    ck = np.arange(10, steps + 1, 10)
    sms = engine.load().tb_num_sms(engine.context(0))
    p = ensemble.pack_ensemble(ham, cfg, 3, range(2 * sms + 40), "01" * (n // 2), tb.TruncationPolicy(chi, 1e-12), ck)
    runs = {}
    for small in ("0", "1"):
        monkeypatch.setenv("TB_SMALL_ENGINE", small)
        runs[small] = ensemble.run_packed(p)
    a, b = runs["0"], runs["1"]
    np.testing.assert_array_equal(a.values, b.values)
    np.testing.assert_array_equal(a.discarded, b.discarded)
    np.testing.assert_array_equal(a.ledger, b.ledger)
    np.testing.assert_array_equal(a.sum_v, b.sum_v)
    np.testing.assert_array_equal(a.sum_v2, b.sum_v2)
    assert a.flops == pytest.approx(b.flops, rel=1e-12)


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
