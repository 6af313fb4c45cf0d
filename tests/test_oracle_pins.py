"""Pin the CPU oracle (oracle/mps_oracle.py) against fixtures produced by the
unmodified reference (tests/golden/make_golden.py).  Same numpy/LAPACK calls
in the same order, so agreement is at rounding level (bitwise in practice)."""

import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from oracle.mps_oracle import OracleMPS, run_sample_checkpoints

DELTA = math.pi / 2**7


def _circ(n, hs, cs, steps, T, i):
    ham = tb.build_spin_ring(n, 1.0, hs)
    return tb.sample_circuit(ham, tb.PaiConfig(DELTA, steps, T), tb.circuit_stream(cs, i), sample_id=i)


@pytest.mark.parametrize("i", [0, 1, 7, 42])
def test_oracle_c1_matches_reference(golden, i):
    ref = golden("ref_c1.npz")
    vals, sign, disc, counters = run_sample_checkpoints(_circ(8, 0, 1, 100, 1.0, i), "01" * 4, 16, 1e-12,
                                                        ref["checkpoints"])
    row = int(np.flatnonzero(ref["full_ids"] == i)[0])
    np.testing.assert_allclose(vals, ref["vals_full"][row], rtol=0, atol=1e-13)
    np.testing.assert_array_equal(sign, ref["sign"][i])
    assert counters[0] == ref["ledger"][i][0] and counters[1] == ref["ledger"][i][1]


def test_oracle_c1_statevector(golden):
    ref = golden("ref_c1.npz")
    circ = _circ(8, 0, 1, 100, 1.0, 3)
    st = OracleMPS("01" * 4)
    st.run(circ.operations(), 16, 1e-12)
    buf_psi = _psi(st)
    assert abs(np.vdot(ref["psi"][3], buf_psi)) == pytest.approx(1.0, abs=1e-12)
    np.testing.assert_allclose(buf_psi, ref["psi"][3], atol=1e-12)


def _psi(st):
    vec = np.ones((1, 1), dtype=complex)
    for s in range(st.n):
        vec = np.tensordot(vec, st.block(s), axes=(-1, 0)).reshape(-1, st.dims[s + 1])
    return vec[:, 0]


def test_oracle_c2_truncated_prefix(golden):
    """Truncated regime: per-sample agreement at checkpoints whose cumulative
    discarded weight is still tiny."""
    ref = golden("ref_c2.npz")
    ck = ref["checkpoints"][:3]
    vals, _, disc, _ = run_sample_checkpoints(_circ(16, 2, 3, 200, 2.0, 0), "01" * 8, 32, 1e-12, ck)
    np.testing.assert_allclose(vals, ref["vals_full"][0][:3], rtol=0, atol=1e-9)
    np.testing.assert_allclose(disc, ref["disc"][0][:3], rtol=1e-6, atol=1e-20)


def test_oracle_kats(golden):
    kat = golden("ref_kat.npz")
    st = OracleMPS("+++")
    c = np.zeros(4)
    st.run([(tb.PauliString.from_label("Z0Z1", 3), math.pi / 2)], 16, 1e-12, c)
    assert abs(st.expect({0: "X"}) - float(kat["zz_x0"])) < 1e-15
    assert tuple(st.dims) == tuple(kat["zz_bonds"])
    ham = tb.build_spin_ring(6, 1.0, 11)
    st = OracleMPS("0+1-0+")
    for k, t in enumerate(ham.terms):
        st.run([(t.pauli, 0.3 + 0.01 * k)], None, 1e-14)
    np.testing.assert_allclose(_psi(st), kat["ring6_psi"], atol=1e-13)
    assert tuple(st.dims) == tuple(kat["ring6_dims"])


def test_oracle_pi_local_equals_full_update_untruncated():
    ham = tb.build_spin_ring(6, 1.0, 5)
    ops = [(t.pauli, math.pi if k % 5 == 0 else 0.2) for k, t in enumerate(ham.terms)]
    a, b = OracleMPS("010101"), OracleMPS("010101")
    a.run(ops, None, 1e-14)
    b.run(ops, None, 1e-14, pi_local=True)
    np.testing.assert_allclose(a.z_profile(), b.z_profile(), atol=1e-12)
    assert abs(abs(np.vdot(_psi(a), _psi(b))) - 1.0) < 1e-12


def _tfim_setup(ref):
    ham = tb.build_tfim_ring(6, 1.0, 6)
    np.testing.assert_array_equal(ham.coefficients(), ref["coeffs"])  # same draw and term order as the fixture
    return ham, tb.PaiConfig(math.pi / 2**6, 40, 0.5)


def test_tfim_builder_conventions():
    ham = tb.build_tfim_ring(8, 1.0, 6)
    labels = [t.pauli.label() for t in ham.terms]
    assert labels[:8] == [tb.PauliString.single(8, k, "Z").label() for k in range(8)]
    assert labels[8:16] == [tb.PauliString.single(8, k, "X").label() for k in range(8)]
    assert [t.pauli.support for t in ham.terms[16:]] == [(b, b + 1) for b in range(7)] + [(0, 7)]
    assert all(0.5 <= t.coeff <= 1.5 for t in ham.terms[16:])
    # config 4 as written is outside the sampler's domain; the first feasible step count is accepted
    big = tb.build_tfim_ring(50, 1.0, 6)
    with pytest.raises(ValueError):
        tb.PaiConfig(math.pi / 2**8, 300, 3.0).validate_against(big)
    n = tb.min_trotter_steps(big, math.pi / 2**8, 3.0)
    tb.PaiConfig(math.pi / 2**8, n, 3.0).validate_against(big)
    with pytest.raises(ValueError):
        tb.PaiConfig(math.pi / 2**8, n - 1, 3.0).validate_against(big)


@pytest.mark.parametrize("i", [0, 5, 11])
def test_oracle_tfim_matches_reference(golden, i):
    ref = golden("ref_tfim_n6.npz")
    ham, cfg = _tfim_setup(ref)
    circ = tb.sample_circuit(ham, cfg, tb.circuit_stream(7, i), sample_id=i)
    vals, sign, _, _ = run_sample_checkpoints(circ, "0" * 6, 8, 1e-12, list(ref["checkpoints"]))
    np.testing.assert_allclose(vals, ref["vals"][i], atol=1e-12)
    np.testing.assert_array_equal(sign, ref["sign"][i])


def test_oracle_tfim_trotter_matches_reference(golden):
    ref = golden("ref_tfim_n6.npz")
    ham, _ = _tfim_setup(ref)
    for chi, key in ((8, "trot_exact"), (4, "trot_trunc")):
        st, done, out = OracleMPS("0" * 6), 0, []
        for j in ref["checkpoints"]:
            st.run(tb.build_trotter_circuit(ham, (j - done) * 0.5 / 40, int(j - done)).operations(), chi, 1e-12)
            done = j
            out.append(st.z_profile())
        np.testing.assert_allclose(np.array(out), ref[key], atol=1e-12)
