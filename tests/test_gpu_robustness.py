"""Failure paths and determinism of the engine (GPU): per-sample exclusion of
a non-converged SVD instead of failing the launch, refusal to continue a slot
whose workspace generation changed, private slot pools per pipeline, the
device-resident step path, and bitwise run-to-run reproducibility."""

import ctypes
import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import _lib, ensemble
from paper_2604_13144_b200.estimator import quantize

pytestmark = pytest.mark.gpu
DELTA = math.pi / 2**7


def _c1():
    return tb.build_spin_ring(8, 1.0, 0), tb.PaiConfig(DELTA, 100, 1.0), np.arange(10, 101, 10)


def test_nonconverged_samples_are_excluded_not_fatal(engine, monkeypatch):
    # fault injection (test hook): every SVD of the samples with index % 5 == 0
    # reports non-convergence
    ham = tb.build_spin_ring(16, 1.0, 2)
    cfg = tb.PaiConfig(DELTA, 30, 0.3)
    ck = np.array([10, 20, 30])
    pol = tb.TruncationPolicy(32, 1e-12)
    monkeypatch.setenv("TB_FAULT_INJECT", "5")
    run = tb.run_ensemble(ham, cfg, 3, range(24), "01" * 8, pol, ck)
    ex = run.excluded
    np.testing.assert_array_equal(ex >= 0, np.arange(24) % 5 == 0)
    counts = run.row_counts()
    np.testing.assert_array_equal(counts, 24 - ensemble.excluded_counts(ex, ck.size))
    # the sums hold exactly the checkpoints before each sample's exclusion point
    p = ensemble.pack_ensemble(ham, cfg, 3, range(24), "01" * 8, pol, ck)
    want = np.zeros_like(run.sum_v)
    for s in range(24):
        stop = ck.size if ex[s] < 0 else ex[s]
        want[:stop] += quantize(p.ckpt_sign[s, :stop, None] * run.values[s, :stop])
    np.testing.assert_array_equal(run.sum_v, want)
    # without the exclusion array the launch fails and the caller's arrays stay untouched
    S, C, O = 24, ck.size, 16
    sv = np.full((C, O), 7, np.int64)
    sv2 = np.full((C, O), 7, np.int64)
    flops = np.zeros(1)
    arrays = [np.ascontiguousarray(x) for x in (p.words, p.offsets, p.ckpt_end, p.ckpt_sign, p.angle_cs, p.weights,
                                                 p.obs_sites, p.init_vecs)]
    w, off, ce, cs, ang, wt, obs, iv = arrays
    desc = _lib.EnsembleDesc(p.n, p.cap, p.chi_cut, 1, p.floor, S, C, O, ang.shape[0], w.ctypes.data,
                             off.ctypes.data, ce.ctypes.data, cs.ctypes.data, ang.ctypes.data, wt.ctypes.data,
                             obs.ctypes.data, iv.ctypes.data, None, None, 0, 0)
    out = _lib.EnsembleOut(None, None, None, sv.ctypes.data, sv2.ctypes.data, flops.ctypes.data, None, None)
    ctx = _lib.context(0)
    rc = _lib.load().tb_run_ensemble(ctx, ctypes.byref(desc), ctypes.byref(out))
    assert rc == -4  # TB_ENOCONV
    assert np.all(sv == 7) and np.all(sv2 == 7) and flops[0] == 0


def test_stale_slot_is_refused(engine):
    ham, cfg, ck = _c1()
    pipe = tb.SlotPipeline(ham, cfg, 1, "01" * 4, tb.TruncationPolicy(16), ck, n_slots=4)
    pipe.step_host(pipe.plan())
    # another engine call on the pipeline's own context reuses (and reallocates) its pool
    a = np.random.default_rng(0).normal(size=(300, 8, 8)) + 0j
    s = np.zeros((300, 8))
    _lib.check(_lib.load().tb_svd(pipe.ctx, a.ctypes.data, 300, 8, 8, s.ctypes.data, None, None), pipe.ctx)
    with pytest.raises(ValueError, match="reset every slot"):
        pipe.step_host(pipe.plan())
    pipe.close()


def test_pipelines_have_private_slot_pools(engine):
    ham, cfg, ck = _c1()
    pol = tb.TruncationPolicy(16)
    a = tb.SlotPipeline(ham, cfg, 1, "01" * 4, pol, ck, n_slots=6)
    b = tb.SlotPipeline(ham, cfg, 1, "01" * 4, pol, ck, n_slots=6, first_sample=100)
    for _ in range(ck.size):  # interleaved steps, plus a drop-in call on the shared context in between
        a.step_host(a.plan())
        st = tb.init_product_state("01" * 4)
        tb.apply_pauli_rotation(st, tb.PauliString.from_label("X0X1", 8), 0.3, pol)
        b.step_host(b.plan())
    ra = tb.run_ensemble(ham, cfg, 1, range(6), "01" * 4, pol, ck)
    rb = tb.run_ensemble(ham, cfg, 1, range(100, 106), "01" * 4, pol, ck)
    np.testing.assert_array_equal(a.sum_v, ra.sum_v)
    np.testing.assert_array_equal(b.sum_v, rb.sum_v)
    a.close()
    b.close()


def test_device_step_path_matches_host_path(engine):
    import torch

    ham, cfg, ck = _c1()
    pol = tb.TruncationPolicy(16)
    host = tb.SlotPipeline(ham, cfg, 1, "01" * 4, pol, ck, n_slots=20)
    host.run(ck.size + 3)
    dev = tb.SlotPipeline(ham, cfg, 1, "01" * 4, pol, ck, n_slots=20)
    ds = dev.device_state()
    stream = torch.cuda.Stream()
    for p in dev.planned(ck.size + 3):
        dev.step_device(dev.upload(p, stream), ds, stream.cuda_stream)
    dev.sync_from_device(ds)
    np.testing.assert_array_equal(dev.sum_v, host.sum_v)
    np.testing.assert_array_equal(dev.sum_v2, host.sum_v2)
    np.testing.assert_array_equal(dev.row_count, host.row_count)
    assert dev.flops == pytest.approx(host.flops, rel=1e-12)
    for c, st in host.stats().items():
        np.testing.assert_array_equal(dev.stats()[c]["estimate"], st["estimate"])


def test_bitwise_reproducible_runs_truncated(engine):
    """Fixed sweep order and fixed-order reductions: two independent runs of a
    truncated (C2-shaped, chi 32) ensemble give bit-identical per-sample
    values and sums (SURVEY.md §7 'Determinism')."""
    ham = tb.build_spin_ring(16, 1.0, 2)
    cfg = tb.PaiConfig(DELTA, 200, 2.0)
    ck = np.arange(10, 201, 10)
    pol = tb.TruncationPolicy(32, 1e-12)
    outs = []
    for _ in range(2):
        pipe = tb.SlotPipeline(ham, cfg, 3, "01" * 8, pol, ck, n_slots=64)
        vals = []
        for p in pipe.planned(ck.size):
            v = np.zeros((64, 1, 16))
            pipe.step_host(p, v)
            vals.append(v)
        outs.append((np.stack(vals), pipe.sum_v.copy(), pipe.sum_v2.copy()))
        pipe.close()
    assert np.array_equal(outs[0][0], outs[1][0])
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][2], outs[1][2])
