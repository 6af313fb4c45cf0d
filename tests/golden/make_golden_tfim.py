"""Golden fixture for the transverse-field Ising ring (config 4 at desk scale),
produced with the UNMODIFIED reference (un-jitted, see make_golden.py).

The reference has no TFIM builder; the Hamiltonian is assembled here from the
reference's own generic ``Hamiltonian``/``HamTerm``/``PauliString`` types
(pauli.py:130-167) with the draw and term order that
``paper_2604_13144_b200.pauli.build_tfim_ring`` documents (J then h from
``disorder_stream(seed)``; Z fields, X fields, ZZ bonds).  Contents:
- ``vals``/``sign``: 16 TE-PAI samples from the all-|0> state, <Z_j> for all j
  at prefix checkpoints, untruncated (chi 8 = 2^(n/2));
- ``trot_exact``/``trot_trunc``: the deterministic first-order Trotter
  circuit at the same time grid, chi 8 and chi 4 (truncation active).

Usage: python tests/golden/make_golden_tfim.py     Writes: tests/golden/ref_tfim_n6.npz
"""
import dataclasses, math, os, sys

os.environ.setdefault("NUMBA_DISABLE_JIT", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np  # noqa: E402
import tepai  # noqa: E402
from tepai import rng as trng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N, HSEED, CSEED, G = 6, 6, 7, 1.0
DELTA, STEPS, T = math.pi / 2**6, 40, 0.5
CKPT = [10, 20, 30, 40]
NS = 16


def tfim(n, g, seed):
    rng = trng.disorder_stream(seed)
    J = rng.uniform(0.5, 1.5, size=n)
    h = rng.uniform(-1.0, 1.0, size=n)
    P = tepai.PauliString
    terms = [tepai.HamTerm(float(h[k]), P.single(n, k, "Z")) for k in range(n) if h[k] != 0.0]
    terms += [tepai.HamTerm(float(g), P.single(n, k, "X")) for k in range(n)]
    terms += [tepai.HamTerm(float(J[b]), P(n, ((b, "Z"), ((b + 1) % n, "Z")))) for b in range(n)]
    return tepai.Hamiltonian(n, tuple(terms), coupling=0.0, seed=seed)


def zs(st):
    return [tepai.expectation(st, tepai.PauliString.single(N, q, "Z")) for q in range(N)]


def trotter(ham, chi):
    pol = tepai.TruncationPolicy(chi_cut=chi, svalue_floor=1e-12)
    st = tepai.init_product_state("0" * N)
    out, done = [], 0
    for j in CKPT:
        tepai.run_circuit(st, tepai.build_trotter_circuit(ham, (j - done) * T / STEPS, j - done), pol)
        done = j
        out.append(zs(st))
    return np.array(out), st.discarded_weight


def main():
    ham = tfim(N, G, HSEED)
    cfg = tepai.PaiConfig(DELTA, STEPS, T)
    cfg.validate_against(ham)
    policy = tepai.TruncationPolicy(chi_cut=8, svalue_floor=1e-12)
    vals = np.zeros((NS, len(CKPT), N))
    sign = np.zeros((NS, len(CKPT)), np.int64)
    for i in range(NS):
        circ = tepai.sample_circuit(ham, cfg, trng.circuit_stream(CSEED, i), sample_id=i)
        st = tepai.init_product_state("0" * N)
        lo = 0
        for c, j in enumerate(CKPT):
            hi = int(np.searchsorted(circ.step_index, j))
            seg = dataclasses.replace(circ, term_index=circ.term_index[lo:hi], step_index=circ.step_index[lo:hi],
                                      kinds=circ.kinds[lo:hi], signs=circ.signs[lo:hi])
            tepai.run_circuit(st, seg, policy)
            lo = hi
            vals[i, c] = zs(st)
            sign[i, c] = 1 - 2 * (int(np.count_nonzero(circ.kinds[:hi] == 2)) & 1)
    te, _ = trotter(ham, 8)
    tt, disc = trotter(ham, 4)
    np.savez_compressed(os.path.join(HERE, "ref_tfim_n6.npz"), vals=vals, sign=sign, checkpoints=np.array(CKPT),
                        coeffs=ham.coefficients(), trot_exact=te, trot_trunc=tt, trot_trunc_discarded=disc)
    print("written", vals.shape, "trunc discarded", disc)


if __name__ == "__main__":
    main()
