"""GPU parity tests: the CUDA engine (through the C ABI) against the CPU oracle
and the reference-generated golden fixtures.

Tolerances (north_star): untruncated <= 1e-10 (absolute on
<Z> in [-1, 1]); truncated regime per sample <= 1e-8 only while the
cumulative discarded weight is tiny; gauge-dependent tensors are compared
through gauge-invariant quantities (expectations, state vectors, singular
values)."""

import math

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from oracle.mps_oracle import OracleMPS, run_sample_checkpoints

pytestmark = pytest.mark.gpu
DELTA = math.pi / 2**7


def _svd_gpu(engine, a):
    lib, ctx = engine.load(), engine.context(0)
    b, m, n = a.shape
    k = min(m, n)
    a = np.ascontiguousarray(a, dtype=np.complex128)
    s = np.zeros((b, k))
    u = np.zeros((b, m, k), np.complex128)
    vh = np.zeros((b, k, n), np.complex128)
    engine.check(lib.tb_svd(ctx, a.ctypes.data, b, m, n, s.ctypes.data, u.ctypes.data, vh.ctypes.data), ctx)
    return u, s, vh


@pytest.mark.parametrize("m,n", [(2, 2), (4, 16), (16, 4), (32, 32), (64, 128), (128, 64), (128, 128), (256, 256)])
def test_jacobi_svd_matches_lapack(engine, m, n):
    _check_svd(engine, m, n)


# chi = 128 shapes (the wide path: block-streamed Jacobi + global-memory QRCP),
# including ragged column blocks, with and without the QR preconditioner
@pytest.mark.parametrize("m,n", [(256, 33), (129, 129), (200, 97), (97, 200), (256, 128), (136, 256)])
@pytest.mark.parametrize("precond", ["0", "1"])
def test_wide_svd_matches_lapack(engine, monkeypatch, m, n, precond):
    monkeypatch.setenv("TB_PRECOND", precond)
    _check_svd(engine, m, n)


# QR preconditioner with the matrix in tensor memory (TB_QRCP_TMEM=1, the
# default) and the shared-memory variant (0): same parity bar on the
# half-warp (<= 128) shapes they serve
@pytest.mark.parametrize("m,n", [(32, 32), (64, 128), (128, 64), (128, 128), (100, 77), (128, 96)])
@pytest.mark.parametrize("tmem", ["0", "1"])
def test_tmem_qrcp_svd_matches_lapack(engine, monkeypatch, m, n, tmem):
    monkeypatch.setenv("TB_QRCP_TMEM", tmem)
    _check_svd(engine, m, n)


# Gram screen of the late Jacobi sweeps (DMMA Gram matrix, flagged pairs only):
# off (0), screened visits (1), + flag-driven cross phases (2, the default);
# shapes with 2..4 column blocks and 64 / 128 rows, ragged ones included
@pytest.mark.parametrize("m,n", [(128, 128), (64, 128), (128, 64), (64, 64), (100, 77), (128, 96), (72, 128)])
@pytest.mark.parametrize("mode", ["0", "1", "2"])
def test_gram_screen_svd_matches_lapack(engine, monkeypatch, m, n, mode):
    monkeypatch.setenv("TB_GRAM_SCREEN", mode)
    _check_svd(engine, m, n)


def _check_svd(engine, m, n):
    rng = np.random.default_rng(m * 1000 + n)
    k = min(m, n)
    # graded spectrum down to 1e-14 plus an exactly rank-deficient tail
    q1, _ = np.linalg.qr(rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k)))
    q2, _ = np.linalg.qr(rng.normal(size=(n, k)) + 1j * rng.normal(size=(n, k)))
    sv = np.logspace(0, -14, k)
    if k >= 8:
        sv[-(k // 8):] = 0.0
    a = np.stack([(q1 * sv) @ q2.conj().T, rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))])
    u, s, vh = _svd_gpu(engine, a)
    for b in range(2):
        ref = np.linalg.svd(a[b], compute_uv=False)
        np.testing.assert_allclose(s[b] / ref[0], ref / ref[0], rtol=0, atol=1e-13)
        rec = (u[b] * s[b]) @ vh[b]
        assert np.linalg.norm(rec - a[b]) <= 1e-12 * np.linalg.norm(a[b])
        live = s[b] > 1e-10 * s[b][0]
        uu = u[b][:, live]
        assert np.abs(uu.conj().T @ uu - np.eye(uu.shape[1])).max() < 1e-12


# truncated splits (tail skipping): only the kcut kept triplets must be those
# of the full SVD; spectrum shaped like a saturated chi=64 bond (kept values
# graded to 1e-10, a tail of ~1e-11 .. 1e-14 values, an exact null space)
@pytest.mark.parametrize("m,n,kcut", [(128, 128, 64), (64, 64, 32), (128, 64, 16), (64, 128, 40), (256, 256, 128),
                                      (200, 256, 100)])
def test_truncated_svd_keeps_exact_triplets(engine, m, n, kcut):
    lib, ctx = engine.load(), engine.context(0)
    rng = np.random.default_rng(7 * m + n + kcut)
    k = min(m, n)
    mats = []
    for b in range(3):
        q1, _ = np.linalg.qr(rng.normal(size=(m, k)) + 1j * rng.normal(size=(m, k)))
        q2, _ = np.linalg.qr(rng.normal(size=(n, k)) + 1j * rng.normal(size=(n, k)))
        sv = np.concatenate([np.logspace(0, -10, kcut), 10.0 ** rng.uniform(-14, -10.5, k - kcut)])
        sv[-(k // 10):] = 0.0
        if b == 2:  # the tail is the whole spectrum's second half at 1e-3: T stays small or empty
            sv[kcut:] = 1e-3 * rng.uniform(size=k - kcut)
        mats.append((q1 * sv) @ q2.conj().T)
    a = np.ascontiguousarray(np.stack(mats))
    s = np.zeros((3, k))
    u = np.zeros((3, m, k), np.complex128)
    vh = np.zeros((3, k, n), np.complex128)
    engine.check(lib.tb_svd_trunc(ctx, a.ctypes.data, 3, m, n, kcut, s.ctypes.data, u.ctypes.data, vh.ctypes.data),
                 ctx)
    for b in range(3):
        uu, ref, vv = np.linalg.svd(a[b], full_matrices=False)
        fro2 = np.linalg.norm(a[b]) ** 2
        np.testing.assert_allclose(s[b, :kcut] / ref[0], ref[:kcut] / ref[0], rtol=0, atol=1e-13)
        assert abs(np.sum(s[b] ** 2) - fro2) <= 1e-12 * fro2
        best = (uu[:, :kcut] * ref[:kcut]) @ vv[:kcut]
        mine = (u[b][:, :kcut] * s[b, :kcut]) @ vh[b][:kcut]
        assert np.linalg.norm(mine - best) <= 1e-12 * np.linalg.norm(a[b])
        live = s[b, :kcut] > 1e-10 * s[b][0]
        ul = u[b][:, :kcut][:, live]
        assert np.abs(ul.conj().T @ ul - np.eye(ul.shape[1])).max() < 1e-12


def test_single_gate_known_answers(engine, golden):
    kat = golden("ref_kat.npz")
    st = tb.init_product_state("+++")
    tb.apply_pauli_rotation(st, tb.PauliString.from_label("Z0Z1", 3), math.pi / 2, tb.TruncationPolicy(16))
    assert abs(tb.expectation(st, tb.PauliString.from_label("X0", 3)) - float(kat["zz_x0"])) < 1e-14
    assert st.bond_dims == tuple(kat["zz_bonds"])
    st = tb.init_product_state("00")
    tb.apply_pauli_rotation(st, tb.PauliString.from_label("X0", 2), math.pi, tb.TruncationPolicy(16))
    assert tb.expectation(st, tb.PauliString.from_label("Z0", 2)) == pytest.approx(-1.0, abs=1e-15)
    # identity-angle gate: state and ledger unchanged
    led = tb.CostLedger()
    before = st.buf.copy()
    tb.apply_pauli_rotation(st, tb.PauliString.from_label("X0X1", 2), 0.0, tb.TruncationPolicy(16), led)
    assert led.gate_count == 0 and np.array_equal(before, st.buf)


def test_ring_swap_network_statevector(engine, golden):
    kat = golden("ref_kat.npz")
    ham = tb.build_spin_ring(6, 1.0, 11)
    st = tb.init_product_state("0+1-0+")
    for k, t in enumerate(ham.terms):
        tb.apply_pauli_rotation(st, t.pauli, 0.3 + 0.01 * k, tb.EXACT)
    assert st.bond_dims == tuple(kat["ring6_dims"])
    np.testing.assert_allclose(st.to_statevector(), kat["ring6_psi"], atol=1e-12)


def test_run_circuit_statevector_vs_reference(engine, golden):
    ref = golden("ref_c1.npz")
    ham = tb.build_spin_ring(8, 1.0, 0)
    cfg = tb.PaiConfig(DELTA, 100, 1.0)
    for i in range(4):
        circ = tb.sample_circuit(ham, cfg, tb.circuit_stream(1, i), sample_id=i)
        st = tb.init_product_state("01" * 4)
        led = tb.CostLedger()
        tb.run_circuit(st, circ, tb.TruncationPolicy(16), led)
        np.testing.assert_allclose(st.to_statevector(), ref["psi"][i], atol=1e-10)
        assert abs(tb.expectation(st, tb.PauliString(8)) - 1.0) < 1e-12  # norm
        # whole-circuit call: the ledger's sum of kept-bond cubes obeys the SPEC bound
        assert led.sum_chi_cubed <= led.gate_count * led.chi_max**3


def test_general_pauli_expectation(engine):
    ham = tb.build_spin_ring(7, 1.0, 2)
    st = tb.init_product_state("0+1-01+")
    ora = OracleMPS("0+1-01+")
    ops = [(t.pauli, 0.37 + 0.05 * k) for k, t in enumerate(ham.terms)]
    tb.run_circuit(st, _OpsCircuit(7, ops), tb.EXACT)
    ora.run(ops, None, 1e-14)
    for label in ("X0", "Y3", "Z6", "X1Y2Z5", "Y0Y6", "Z0Z1Z2Z3Z4Z5Z6"):
        p = tb.PauliString.from_label(label, 7)
        assert tb.expectation(st, p) == pytest.approx(ora.expect(dict((s, y) for s, y in p.ops)), abs=1e-12)


class _OpsCircuit:
    def __init__(self, n, ops):
        self.n, self._ops = n, ops

    def operations(self):
        return iter(self._ops)


def test_rank_deficient_centre_move_zero_padded(engine):
    """2*cl < cr on a centre move: the reference fails in a reshape
    (_kernel.py:75); both the oracle and the engine zero-pad."""
    rng = np.random.default_rng(5)
    dims = [1, 1, 4, 2, 1]
    st = tb.MPSState(4)
    st.ensure_capacity(4)
    st.dims = np.array(dims, np.int64)
    ora = OracleMPS("0000")
    ora.grow(4)
    ora.dims = np.array(dims, np.int64)
    for s in range(4):
        t = rng.normal(size=(dims[s], 2, dims[s + 1])) + 1j * rng.normal(size=(dims[s], 2, dims[s + 1]))
        st.buf[s, : dims[s], :, : dims[s + 1]] = t
        ora.buf[s, : dims[s], :, : dims[s + 1]] = t
    nrm = math.sqrt(abs(tb.expectation(st, tb.PauliString(4))))
    st.buf[0] /= nrm
    ora.buf[0] /= nrm
    ops = [(tb.PauliString.from_label("X2Y3", 4), 0.4)]
    tb.run_circuit(st, _OpsCircuit(4, ops), tb.TruncationPolicy(4, 1e-14))
    ora.run(ops, 4, 1e-14)
    for j in range(4):
        p = tb.PauliString.single(4, j, "Z")
        assert tb.expectation(st, p) == pytest.approx(ora.expect({j: "Z"}), abs=1e-12)


@pytest.mark.parametrize("pi_local", [False, True])
def test_c1_ensemble_per_sample_parity(engine, golden, pi_local):
    """Config 1 (untruncated): every sample, every checkpoint, every site vs the
    reference run on the same gate lists, <= 1e-10."""
    ref = golden("ref_c1.npz")
    ham = tb.build_spin_ring(8, 1.0, 0)
    cfg = tb.PaiConfig(DELTA, 100, 1.0)
    ids = ref["full_ids"][:64]
    run = tb.run_ensemble(ham, cfg, 1, ids, "01" * 4, tb.TruncationPolicy(16), ref["checkpoints"], pi_local=pi_local)
    np.testing.assert_allclose(run.values, ref["vals_full"][: len(ids)], rtol=0, atol=1e-10)
    if not pi_local:
        np.testing.assert_array_equal(run.ledger[:, 0], ref["ledger"][: len(ids), 0])
        np.testing.assert_array_equal(run.ledger[:, 1], ref["ledger"][: len(ids), 1])
    # fused fixed-point sums == host quantisation of sign * <Z>
    signs = ref["sign"][: len(ids)].astype(np.float64)
    want_v = tb.estimator.quantize(signs[:, :, None] * run.values).sum(axis=0)
    want_v2 = tb.estimator.quantize(run.values**2).sum(axis=0)
    np.testing.assert_array_equal(run.sum_v, want_v)
    np.testing.assert_array_equal(run.sum_v2, want_v2)


def test_c1_estimator_vs_reference_mean(engine, golden):
    """1,000-sample Z_0 estimate equals the mean of the reference's per-sample
    signed, weighted values (same circuits) to 1e-10."""
    ref = golden("ref_c1.npz")
    ham = tb.build_spin_ring(8, 1.0, 0)
    cfg = tb.PaiConfig(DELTA, 100, 1.0)
    run = tb.run_ensemble(ham, cfg, 1, range(1000), "01" * 4, tb.TruncationPolicy(16), ref["checkpoints"],
                          observables=[0], keep_values=True)
    st = run.stats()
    want = ref["weights"] * np.mean(ref["sign"] * ref["z0"], axis=0)
    np.testing.assert_allclose(st["estimate"][:, 0], want, atol=1e-10)
    np.testing.assert_allclose(run.values[:, :, 0], ref["z0"], atol=1e-10)


@pytest.mark.parametrize("tmem", ["0", "1"])
def test_c2_truncated_prefix_parity(engine, golden, monkeypatch, tmem):
    monkeypatch.setenv("TB_QRCP_TMEM", tmem)
    ref = golden("ref_c2.npz")
    ham = tb.build_spin_ring(16, 1.0, 2)
    cfg = tb.PaiConfig(DELTA, 200, 2.0)
    ck = ref["checkpoints"][:4]
    run = tb.run_ensemble(ham, cfg, 3, range(4), "01" * 8, tb.TruncationPolicy(32, 1e-12), ck, pi_local=False)
    for i in range(4):
        ok = ref["disc"][i][:4] < 1e-7
        np.testing.assert_allclose(run.values[i][ok], ref["vals_full"][i][:4][ok], atol=1e-8)
        # cumulative discarded weight: (total - kept)/total per update carries
        # ~1e-16 cancellation noise in the reference's own formula
        # (_kernel.py:130) and near-degenerate cut values make the per-update
        # weights chaotic once truncation bites, so it is matched to 25 %
        np.testing.assert_allclose(run.discarded[i][ok], ref["disc"][i][:4][ok], rtol=0.25, atol=1e-13)


@pytest.mark.parametrize("tmem", ["0", "1"])
def test_c3_headline_prefix_parity(engine, golden, monkeypatch, tmem):
    monkeypatch.setenv("TB_QRCP_TMEM", tmem)
    ref = golden("ref_c3.npz")
    ham = tb.build_spin_ring(32, 1.0, 4)
    cfg = tb.PaiConfig(DELTA, 200, 2.0)
    ck = ref["checkpoints"]
    run = tb.run_ensemble(ham, cfg, 5, range(2), "01" * 16, tb.TruncationPolicy(64, 1e-12), ck, pi_local=False)
    for i in range(2):
        np.testing.assert_allclose(run.values[i], ref["vals_full"][i], atol=1e-8)
        np.testing.assert_allclose(run.discarded[i], ref["disc"][i], rtol=0.25, atol=1e-13)


def test_empty_and_degenerate_inputs(engine):
    st = tb.init_product_state("0101")
    before = st.tensors
    tb.run_circuit(st, _OpsCircuit(4, []), tb.TruncationPolicy(4))
    assert all(np.array_equal(x, y) for x, y in zip(before, st.tensors)) and st.bond_dims == (1,) * 5
    ham = tb.build_spin_ring(4, 1.0, 0)
    cfg = tb.PaiConfig(DELTA, 5, 0.0)  # T = 0: no non-identity draws
    run = tb.run_ensemble(ham, cfg, 0, range(3), "0101", tb.TruncationPolicy(4), [5])
    np.testing.assert_allclose(run.values[:, 0, :], np.tile([1, -1, 1, -1], (3, 1)), atol=0)
    run = tb.run_ensemble(ham, tb.PaiConfig(DELTA, 10, 0.1), 0, [], "0101", tb.TruncationPolicy(4), [5])
    assert run.n_samples == 0


@pytest.mark.parametrize("slots", [12, 300])
def test_slot_pipeline_matches_whole_circuit_runs(engine, golden, slots):
    """Continuous batching (tb_step, one checkpoint segment per launch, slots
    restarted with new sample ids) gives the same estimator sums as
    tb_run_ensemble over the same ids (bench.py's step definition); 300 slots
    exceed the SM count, so slots queue onto the persistent CTAs and a slot's
    state moves between CTAs from one launch to the next."""
    ref = golden("ref_c1.npz")
    ham = tb.build_spin_ring(8, 1.0, 0)
    cfg = tb.PaiConfig(DELTA, 100, 1.0)
    ck = ref["checkpoints"]
    pipe = tb.SlotPipeline(ham, cfg, 1, "01" * 4, tb.TruncationPolicy(16), ck, n_slots=slots, pi_local=False)
    per_sample = {}
    for _ in range(2 * ck.size):  # two full circuits per slot: ids 0 .. 2 slots - 1
        plan = pipe.plan()
        vals = np.zeros((pipe.n_slots, 1, 8))
        ids = [pipe.slot_pack[b] for b in range(pipe.n_slots)]
        pipe.step_host(plan, vals)
        for b in range(pipe.n_slots):
            per_sample.setdefault(id(ids[b]), []).append(vals[b, 0])
    assert pipe.completed == 2 * slots
    run = tb.run_ensemble(ham, cfg, 1, range(2 * slots), "01" * 4, tb.TruncationPolicy(16), ck, pi_local=False)
    np.testing.assert_array_equal(pipe.sum_v, run.sum_v)
    np.testing.assert_array_equal(pipe.sum_v2, run.sum_v2)
    np.testing.assert_array_equal(pipe.row_count, np.full(ck.size, 2 * slots))
    st = pipe.stats()
    np.testing.assert_allclose(st[ck.size - 1]["estimate"], run.stats()["estimate"][-1], atol=1e-15)


def test_chi128_bonds_vs_oracle(engine):
    """chi = 128 (the C5 bond capacity): 256x256 two-site problems run on the
    L2-resident Jacobi path; brickwork of generic rotations on n = 16 grows the
    centre bond past 64, untruncated (cap = 128 > reached bonds) vs the oracle."""
    n = 16
    rng = np.random.default_rng(3)
    ops = []
    for layer in range(8):
        for a in range(layer % 2, n - 1, 2):
            for sym in "XYZ":
                ops.append((tb.PauliString(n, ((a, sym), (a + 1, sym))), float(rng.uniform(0.3, 1.2))))
    st = tb.init_product_state("01" * 8)
    ora = OracleMPS("01" * 8)
    pol = tb.TruncationPolicy(128, 1e-14)
    tb.run_circuit(st, _OpsCircuit(n, ops), pol)
    ora.run(ops, 128, 1e-14)
    assert max(st.bond_dims) > 64
    assert st.bond_dims == tuple(int(d) for d in ora.dims)
    for j in (0, 5, 8, 15):
        p = tb.PauliString.single(n, j, "Z")
        assert tb.expectation(st, p) == pytest.approx(ora.expect({j: "Z"}), abs=1e-10)


def test_hybrid_trotter_then_tepai_vs_reference(engine, golden):
    """Config 5 schedule at desk scale: Trotter evolution on the GPU
    (continuous angles through tb_run_stream) to t0, then 16 TE-PAI samples
    that all start from that MPS (init_mps fan-out), vs the reference."""
    ref = golden("ref_hybrid_n6.npz")
    ham = tb.build_spin_ring(6, 1.0, 8)
    cfg = tb.PaiConfig(math.pi / 2**6, 20, 0.4)
    run, st0 = tb.run_hybrid(ham, 30, 0.6, cfg, 9, range(16), "010101", tb.TruncationPolicy(8, 1e-12),
                             ref["checkpoints"], pi_local=False)
    np.testing.assert_allclose(st0.to_statevector(), ref["psi_t0"], atol=1e-11)
    np.testing.assert_allclose(run.values, ref["vals"], atol=1e-10)
    signs = ref["sign"].astype(np.float64)
    want = tb.estimator.quantize(signs[:, :, None] * ref["vals"]).sum(axis=0)
    assert np.max(np.abs(run.sum_v - want)) <= 16  # 2^-40 quantisation of values equal to 1e-10


def test_tfim_ensemble_and_trotter_vs_reference(engine, golden):
    """Config 4 physics at desk scale (tests/golden/make_golden_tfim.py): the
    transverse-field Ising ring has non-diagonal X-field one-site gates and
    Z_bZ_{b+1} couplings; 16 TE-PAI samples from |000000> untruncated, and the
    deterministic Trotter circuit on the same kernels at chi 8 (exact) and
    chi 4 (truncation active, discarded weight ~1.7e-8)."""
    ref = golden("ref_tfim_n6.npz")
    ham = tb.build_tfim_ring(6, 1.0, 6)
    np.testing.assert_array_equal(ham.coefficients(), ref["coeffs"])
    cfg = tb.PaiConfig(math.pi / 2**6, 40, 0.5)
    ck = [int(j) for j in ref["checkpoints"]]
    run = tb.run_ensemble(ham, cfg, 7, range(16), "0" * 6, tb.TruncationPolicy(8, 1e-12), ck, pi_local=False)
    np.testing.assert_allclose(run.values, ref["vals"], atol=1e-10)
    run_pi = tb.run_ensemble(ham, cfg, 7, range(16), "0" * 6, tb.TruncationPolicy(8, 1e-12), ck, pi_local=True)
    np.testing.assert_allclose(run_pi.values, ref["vals"], atol=1e-10)
    for chi, key, tol in ((8, "trot_exact", 1e-10), (4, "trot_trunc", 1e-8)):
        st, done, out = tb.init_product_state("0" * 6), 0, []
        for j in ck:
            tb.run_circuit(st, tb.build_trotter_circuit(ham, (j - done) * 0.5 / 40, j - done),
                           tb.TruncationPolicy(chi, 1e-12))
            done = j
            out.append([tb.expectation(st, tb.PauliString.single(6, q, "Z")) for q in range(6)])
        np.testing.assert_allclose(np.array(out), ref[key], atol=tol)
    if chi == 4:
        assert st.discarded_weight == pytest.approx(float(ref["trot_trunc_discarded"]), rel=1e-6)
