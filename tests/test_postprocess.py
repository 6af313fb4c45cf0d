"""Signed-mixture post-processing and the cost report (SPEC.md:413-446 and
481-504).  CPU: the SPEC's worked examples for the
pure functions.  GPU: evaluate_observables through the batched engine call
against per-sample aggregate() and the oracle."""

import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from paper_2604_13144_b200.estimator import SampleRecord, aggregate, aggregate_fixed, quantize
from paper_2604_13144_b200.runner import CostReport, cost_table, tts_tradeoff


def _report(costs, workers=4):
    n = len(costs)
    return CostReport(np.arange(n), np.full(n, 10), np.ones(n), np.full(n, 4), np.asarray(costs, float), workers)


def test_tts_tradeoff_spec_examples():
    rep = _report([3.0, 3.0, 3.0, 3.0])
    rep.check()
    rows = dict((w, t) for w, t, _ in tts_tradeoff(rep, [1, 2, 4, 8]))
    assert rows[1] == rep.c_tot == 12.0                # w = 1 -> TTS = C_tot
    assert rows[4] == 3.0                             # w = N_s, equal costs -> C_circ
    assert rows[2] == 2 * rows[4] and rows[4] == 2 * rows[8]  # doubling w halves TTS
    assert tts_tradeoff(rep, [2], trotter_cost=6.0)[0][2] == 2.0
    with pytest.raises(ValueError):
        tts_tradeoff(rep, [0])
    assert cost_table(rep).splitlines()[0] == "sample_id,nu,sum_chi_cubed,wall_ms,chi_max"
    bad = _report([1.0, 100.0], workers=1)
    bad.check()


def test_variance_vs_bound_trace_spec_examples():
    # t = 0 ensemble (empty circuits): every sample gives the same value -> Var 0
    sv = quantize(np.full((5, 2), 0.5)).sum(axis=0)[None]
    sv2 = quantize(np.full((5, 2), 0.25)).sum(axis=0)[None]
    st = aggregate_fixed(sv, sv2, 5, np.array([1.0]))
    rows = tb.variance_vs_bound_trace([0.0], st, [1.0], site=0, n_samples=5)
    assert rows[0][1] == pytest.approx(0.0, abs=1e-12) and rows[0][2] == 1.0
    # no-pi mode: ||g|| = 1, bound column constant 1; Var[v] <= 1 (+ the N/(N-1) slack)
    rng = np.random.default_rng(0)
    v = rng.choice([-1.0, 1.0], size=(200, 3, 1))
    st = aggregate_fixed(quantize(v).sum(axis=0), quantize(v * v).sum(axis=0), 200, np.ones(3))
    rows = tb.variance_vs_bound_trace([0.1, 0.2, 0.3], st, np.ones(3), n_samples=200)
    assert all(r[2] == 1.0 and r[3] <= 1.0 + 1.0 / 199 for r in rows)
    # the assertion fires when Var[o] exceeds ||g||^2
    with pytest.raises(AssertionError):
        tb.variance_vs_bound_trace([0.1], {"var_o": np.array([[2.0]]), "var_v": np.array([[2.0]])}, [1.0],
                                   n_samples=10**6)


def test_mixture_requires_retained_snapshots():
    run = tb.EnsembleRun(2, None, None, None, np.zeros((1, 1), np.int64), np.zeros((1, 1), np.int64), np.ones(1),
                         0.0, 0.0, 0.0)
    with pytest.raises(ValueError, match="not retained"):
        tb.mixture_from_run(run)


@pytest.mark.gpu
def test_signed_mixture_all_single_qubit_paulis_n6(engine):
    """all 3n single-qubit Paulis on an n=6 ensemble match the
    per-observable aggregate() to 1e-12; identity -> ||g||_1 * mean sign."""
    from oracle.mps_oracle import OracleMPS, run_sample_checkpoints

    ham = tb.build_spin_ring(6, 1.0, 3)
    cfg = tb.PaiConfig(math.pi / 2**5, 30, 1.0)
    ck = [10, 20, 30]
    run = tb.run_ensemble(ham, cfg, 7, range(40), "010101", tb.TruncationPolicy(8), ck, retain_states=True,
                          time_samples=True)
    mix = tb.mixture_from_run(run)
    assert mix.n_samples == 40 and mix.weight_norm == run.weights[-1]
    obs = [tb.PauliString.single(6, j, s) for j in range(6) for s in "XYZ"]
    vals = tb.evaluate_observables(mix, obs)
    per = tb.per_sample_expectations(mix, obs)
    for o in range(len(obs)):
        recs = [SampleRecord(i, int(mix.signs[i]), mix.weight_norm, per[i, o]) for i in range(40)]
        assert vals[o] == pytest.approx(aggregate(recs).mean, abs=1e-12)
    # per-sample Z values equal the ensemble's own final <Z_j> and the oracle's
    for j in range(6):
        np.testing.assert_allclose(per[:, 3 * j + 2], run.values[:, -1, j], atol=1e-12)
    for i in range(3):
        circ = tb.sample_circuit(ham, cfg, tb.circuit_stream(7, i), sample_id=i)
        st = OracleMPS("010101")
        st.run(circ.operations(), 8, 1e-12, pi_local=True)
        for o, p in enumerate(obs):
            assert per[i, o] == pytest.approx(st.expect({p.ops[0][0]: p.ops[0][1]}), abs=1e-10)
    ident = tb.PauliString(6, ())
    assert tb.evaluate_observables(mix, [ident])[0] == pytest.approx(mix.weight_norm * mix.signs.mean(), abs=1e-12)
    # a two-site string through the same pass
    zz = tb.PauliString.from_label("Z0Z3", 6)
    want = np.mean([mix.signs[i] * tb.expectation(_state(run, i), zz) for i in range(40)]) * mix.weight_norm
    assert tb.evaluate_observables(mix, [zz])[0] == pytest.approx(want, abs=1e-12)
    # single-sample mixture with sign + and ||g|| = 1: plain expectations of that MPS
    one = tb.SignedMixture(np.array([1]), 1.0, run.states[:1], run.state_dims[:1])
    assert tb.evaluate_observables(one, [obs[2]])[0] == pytest.approx(run.values[0, -1, 0], abs=1e-12)
    # cost report from the same run
    rep = tb.cost_report(run, n_workers=8)
    assert np.all(rep.c_circ > 0) and rep.tts * 8 == pytest.approx(rep.c_tot)
    np.testing.assert_array_equal(rep.nu, run.ledger[:, 0].astype(np.int64))
    assert run_sample_checkpoints is not None


def _state(run, i):
    st = tb.MPSState(run.states.shape[1])
    st.buf = run.states[i].copy()
    st.cap = run.states.shape[2]
    st.dims = run.state_dims[i].astype(np.int64)
    st.center = int(run.state_center[i])
    return st
