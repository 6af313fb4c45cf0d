"""GPU parity of the 8-CTA cluster Jacobi (jacobi_cluster: the chi = 128
two-site problems held in distributed shared memory, SURVEY.md §8 north_star
(1)) against LAPACK and against the single-CTA wide path.

  * tb_svd with TB_CLUSTER=1: one 8-CTA cluster per matrix; singular values,
    reconstruction and orthonormality at the same tolerances as the
    single-CTA SVD tests (graded spectra down to 1e-14 with an exactly
    rank-deficient tail, and dense random matrices), ragged column blocks
    included;
  * tb_run_stream (run_circuit) at cap 128, where the cluster path is the
    default: chi = 128 brickwork vs the oracle (untruncated) and a truncated
    chi = 128 ring circuit vs the single-CTA engine (TB_CLUSTER=0) — both are
    exact SVDs to rounding, so their truncated results agree to ~1e-10;
  * the ensemble in cluster mode (TB_CLUSTER_ENSEMBLE=1) vs the per-SM mode.
"""

import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from oracle.mps_oracle import OracleMPS

from test_gpu_parity import _OpsCircuit, _check_svd

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n", [(256, 256), (256, 33), (129, 129), (200, 97), (97, 200), (136, 256), (256, 17),
                                 (160, 250)])
@pytest.mark.parametrize("precond", ["0", "1"])
def test_cluster_svd_matches_lapack(engine, monkeypatch, m, n, precond):
    monkeypatch.setenv("TB_CLUSTER", "1")
    monkeypatch.setenv("TB_PRECOND", precond)
    _check_svd(engine, m, n)


@pytest.fixture(scope="module")
def brickwork():
    """Nine brickwork layers of generic XX/YY/ZZ rotations on n = 16: the
    centre bonds saturate at cap = 128 (256x256 two-site problems, truncation
    at the cap); the oracle (numpy LAPACK) result is computed once."""
    n = 16
    rng = np.random.default_rng(5)
    ops = []
    for layer in range(9):
        for a in range(layer % 2, n - 1, 2):
            for sym in "XYZ":
                ops.append((tb.PauliString(n, ((a, sym), (a + 1, sym))), float(rng.uniform(0.3, 1.2))))
    ora = OracleMPS("01" * 8)
    ora.run(ops, 128, 1e-14)
    return n, ops, ora


@pytest.mark.parametrize("cluster", ["0", "1"])
def test_chi128_brickwork_cluster_vs_oracle(engine, monkeypatch, brickwork, cluster):
    monkeypatch.setenv("TB_CLUSTER", cluster)
    n, ops, ora = brickwork
    st = tb.init_product_state("01" * 8)
    tb.run_circuit(st, _OpsCircuit(n, ops), tb.TruncationPolicy(128, 1e-14))
    assert max(st.bond_dims) == 128
    assert st.bond_dims == tuple(int(d) for d in ora.dims)
    assert st.discarded_weight == pytest.approx(ora.discarded_weight, rel=1e-6, abs=1e-15)
    for j in (0, 5, 7, 8, 15):
        p = tb.PauliString.single(n, j, "Z")
        assert tb.expectation(st, p) == pytest.approx(ora.expect({j: "Z"}), abs=1e-10)
    x = tb.PauliString(n, ((6, "X"), (7, "Y"), (9, "Z")))
    assert tb.expectation(st, x) == pytest.approx(ora.expect({6: "X", 7: "Y", 9: "Z"}), abs=1e-10)


def test_chi128_truncated_ring_cluster_vs_single_cta(engine, monkeypatch):
    """Truncation active at chi = 96 < the bonds a ring circuit reaches (wide
    256-row problems with 192-column cuts), cluster vs single-CTA engine."""
    n = 16
    ham = tb.build_spin_ring(n, 1.0, 8)
    circ = tb.build_trotter_circuit(ham, 0.6, 12)
    out = {}
    for cl in ("0", "1"):
        monkeypatch.setenv("TB_CLUSTER", cl)
        st = tb.init_product_state("01" * 8)
        tb.run_circuit(st, circ, tb.TruncationPolicy(96, 1e-12))
        out[cl] = (st.bond_dims, st.discarded_weight,
                   [tb.expectation(st, tb.PauliString.single(n, j, "Z")) for j in range(n)])
    assert max(out["1"][0]) == 96
    assert out["1"][0] == out["0"][0]
    assert out["1"][1] == pytest.approx(out["0"][1], rel=1e-6, abs=1e-14)
    np.testing.assert_allclose(out["1"][2], out["0"][2], atol=1e-9)


def test_cluster_ensemble_matches_per_sm_ensemble(engine, monkeypatch):
    n = 16
    ham = tb.build_spin_ring(n, 1.0, 3)
    cfg = tb.PaiConfig(math.pi / 2**6, 50, 1.0)
    ck = [10, 20, 30, 40, 50]
    runs = {}
    for cl in ("0", "1"):
        monkeypatch.setenv("TB_CLUSTER_ENSEMBLE", cl)
        runs[cl] = tb.run_ensemble(ham, cfg, 11, range(6), "01" * 8, tb.TruncationPolicy(128, 1e-12), ck,
                                   pi_local=False)
    assert runs["1"].ledger[:, 2].max() > 64  # the wide (256-row) problems were reached
    np.testing.assert_allclose(runs["1"].values, runs["0"].values, atol=1e-10)
    np.testing.assert_array_equal(runs["1"].ledger[:, 0], runs["0"].ledger[:, 0])
