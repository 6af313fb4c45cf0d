"""Host-side drop-in pieces vs the reference (CPU): Hamiltonian term order,
disorder draw, gamma/probability known answers, and bit-identity of sampled
gate lists against digests produced by the reference sampler itself."""

import hashlib
import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb

DELTA = math.pi / 2**7
CONFIGS = {"c1": (8, 0, 1, 100, 1.0), "c2": (16, 2, 3, 200, 2.0), "c3": (32, 4, 5, 200, 2.0),
           "c5tepai": (32, 8, 9, 100, 1.0)}


def digest(c):
    h = hashlib.sha1()
    for arr in (c.term_index, c.step_index, c.kinds, c.signs):
        h.update(np.ascontiguousarray(arr).tobytes())
    h.update(f"{c.overall_sign} {c.weight_norm!r}".encode())
    return h.hexdigest()


@pytest.mark.parametrize("name,count", [("c1", 200), ("c2", 64), ("c3", 24), ("c5tepai", 16)])
def test_sampler_bit_identical_to_reference(golden, name, count):
    ref = golden("sampler_digests.npz")
    n, hs, cs, steps, T = CONFIGS[name]
    ham = tb.build_spin_ring(n, 1.0, hs)
    np.testing.assert_array_equal(ham.coefficients()[:n], ref[name + "_fields"])
    cfg = tb.PaiConfig(DELTA, steps, T)
    got = [digest(tb.sample_circuit(ham, cfg, tb.circuit_stream(cs, i), sample_id=i)) for i in range(count)]
    assert got == list(ref[name][:count])


def test_spin_ring_structure():
    ham = tb.build_spin_ring(4, 1.0, [0.0] * 4)
    assert ham.num_terms == 12
    labels = [t.pauli.label() for t in ham.terms]
    assert labels[-3:] == ["X0X3", "Y0Y3", "Z0Z3"]
    ham = tb.build_spin_ring(32, 1.0, 4)
    assert ham.num_terms == 128
    np.testing.assert_allclose(ham.coefficients()[:4], [0.2975, 0.1208, 0.0061, -0.5437], atol=1e-4)
    with pytest.raises(ValueError):
        tb.build_spin_ring(2, 1.0, 0)


def test_gamma_known_answers(golden):
    kat = golden("ref_kat.npz")
    np.testing.assert_allclose(tb.gamma_coeffs(math.pi / 4, math.pi / 2), kat["gamma"], rtol=0, atol=0)
    np.testing.assert_allclose(tb.variant_probabilities(math.pi / 4, math.pi / 2), kat["probs"], rtol=0, atol=0)
    assert abs(sum(tb.gamma_coeffs(0.01, 0.03)) - 1.0) < 1e-15
    assert math.isclose(tb.overhead_norm_inf(math.pi / 2, 1, 1), math.e**2)
    assert math.isclose(tb.expected_gate_count_inf(math.pi / 2, 1, 1), 3.0)


def test_config_validation():
    ham = tb.build_spin_ring(8, 1.0, 0)
    with pytest.raises(ValueError):
        tb.PaiConfig(0.0, 10, 1.0)
    with pytest.raises(ValueError):
        tb.sample_circuit(ham, tb.PaiConfig(1e-3, 10, 1.0), tb.circuit_stream(0, 0))


def test_checkpoint_weights_match_reference(golden):
    for name in ("c1", "c2", "c3"):
        ref = golden(f"ref_{name}.npz")
        n, hs, cs, steps, T = CONFIGS[name]
        ham = tb.build_spin_ring(n, 1.0, hs)
        w = tb.checkpoint_weights(ham, tb.PaiConfig(DELTA, steps, T), ref["checkpoints"])
        np.testing.assert_allclose(w, ref["weights"], rtol=1e-15)


def test_grid_and_runs_methods_both_supported():
    ham = tb.build_spin_ring(8, 1.0, 0)
    cfg = tb.PaiConfig(DELTA, 100, 1.0)
    a = tb.sample_circuit(ham, cfg, tb.circuit_stream(1, 0), method="grid")
    b = tb.sample_circuit(ham, cfg, tb.circuit_stream(1, 0), method="runs")
    assert a.nu > 0 and b.nu > 0
    assert np.all(np.diff(a.step_index) >= 0) and np.all(np.diff(b.step_index) >= 0)
