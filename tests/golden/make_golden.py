"""Generate the committed golden fixtures by running the UNMODIFIED reference
``tepai`` package (``/root/reference/pkg/src``) in this container.

The reference's numba kernel does not compile under numba 0.65 (SURVEY.md §0
fact 4), so it runs un-jitted (``NUMBA_DISABLE_JIT=1``): pure Python + numpy
LAPACK, exactly the reference's ``.py_func`` arithmetic.  Checkpoints follow
the prefix semantics of SURVEY.md §8(a): the circuit is run segment by
segment (one ``run_circuit`` call per checkpoint interval, entries with
``step_index`` in [prev, j)), and <Z_q> is read with the reference's own
``expectation`` after each segment.

Usage:  python tests/golden/make_golden.py            (≈5 min on 8 cores)
Writes: tests/golden/*.npz
"""

from __future__ import annotations

import dataclasses
import hashlib
import math
import os
import sys

os.environ.setdefault("NUMBA_DISABLE_JIT", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402
import tepai  # noqa: E402
from tepai import rng as trng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
DELTA = math.pi / 2**7

CONFIGS = {
    # name: (n, ham_seed, circ_seed, n_steps, T, chi)
    "c1": (8, 0, 1, 100, 1.0, 16),
    "c2": (16, 2, 3, 200, 2.0, 32),
    "c3": (32, 4, 5, 200, 2.0, 64),
    "c5tepai": (32, 8, 9, 100, 1.0, 128),
}


def circuit_digest(c) -> str:
    h = hashlib.sha1()
    for arr in (c.term_index, c.step_index, c.kinds, c.signs):
        h.update(np.ascontiguousarray(arr).tobytes())
    h.update(f"{c.overall_sign} {c.weight_norm!r}".encode())
    return h.hexdigest()


def segment(c, lo, hi):
    return dataclasses.replace(c, term_index=c.term_index[lo:hi], step_index=c.step_index[lo:hi],
                               kinds=c.kinds[lo:hi], signs=c.signs[lo:hi])


def run_member(args):
    name, sid, n_ckpt, every, want_state = args
    n, hs, cs, steps, T, chi = CONFIGS[name]
    ham = tepai.build_spin_ring(n, 1.0, hs)
    cfg = tepai.PaiConfig(DELTA, steps, T)
    circ = tepai.sample_circuit(ham, cfg, trng.circuit_stream(cs, sid), sample_id=sid)
    state = tepai.init_product_state("01" * (n // 2))
    policy = tepai.TruncationPolicy(chi_cut=chi, svalue_floor=1e-12)
    ledger = tepai.CostLedger()
    zs = [tepai.PauliString.single(n, q, "Z") for q in range(n)]
    vals = np.zeros((n_ckpt, n))
    disc = np.zeros(n_ckpt)
    sign = np.zeros(n_ckpt, np.int64)
    chi_seen = np.zeros(n_ckpt, np.int64)
    lo = 0
    for ci in range(n_ckpt):
        j = (ci + 1) * every
        hi = int(np.searchsorted(circ.step_index, j, side="left"))
        tepai.run_circuit(state, segment(circ, lo, hi), policy, ledger)
        lo = hi
        vals[ci] = [tepai.expectation(state, z) for z in zs]
        disc[ci] = tepai.discarded_weight(state)
        sign[ci] = 1 - 2 * (int(np.count_nonzero(circ.kinds[:hi] == 2)) & 1)
        chi_seen[ci] = tepai.max_bond(state)
    out = dict(vals=vals, disc=disc, sign=sign, chi=chi_seen,
               ledger=np.array([ledger.gate_count, ledger.sum_chi_cubed, ledger.chi_max], np.float64),
               dims=np.array(state.dims), weight=circ.weight_norm)
    if want_state:
        out["psi"] = state.to_statevector()
    return name, sid, out


def weights(name, n_ckpt, every):
    n, hs, cs, steps, T, chi = CONFIGS[name]
    ham = tepai.build_spin_ring(n, 1.0, hs)
    return np.array([tepai.sampling.circuit_weight_norm(ham, tepai.PaiConfig(DELTA, (c + 1) * every, (c + 1) * every * T / steps))
                     for c in range(n_ckpt)])


def main():
    from multiprocessing import Pool

    digests = {}
    for name, count in (("c1", 1000), ("c2", 64), ("c3", 64), ("c5tepai", 16)):
        n, hs, cs, steps, T, chi = CONFIGS[name]
        ham = tepai.build_spin_ring(n, 1.0, hs)
        cfg = tepai.PaiConfig(DELTA, steps, T)
        digests[name] = np.array([circuit_digest(tepai.sample_circuit(ham, cfg, trng.circuit_stream(cs, i), sample_id=i))
                                  for i in range(count)])
        digests[name + "_fields"] = ham.coefficients()[:n]
    np.savez_compressed(os.path.join(HERE, "sampler_digests.npz"), **digests)

    jobs = [("c1", i, 10, 10, i < 8) for i in range(1000)]
    jobs += [("c2", i, 20, 10, False) for i in range(4)]
    jobs += [("c3", i, 3, 10, False) for i in range(2)]
    with Pool(os.cpu_count()) as pool:
        res = pool.map(run_member, jobs, chunksize=1)
    by = {}
    for name, sid, out in res:
        by.setdefault(name, {})[sid] = out
    for name, members in by.items():
        ids = sorted(members)
        keep_full = ids if name != "c1" else ids[:200]
        every = 10
        n_ckpt = members[ids[0]]["vals"].shape[0]
        payload = dict(
            sample_ids=np.array(ids),
            vals_full=np.stack([members[i]["vals"] for i in keep_full]),
            full_ids=np.array(keep_full),
            z0=np.stack([members[i]["vals"][:, 0] for i in ids]),
            disc=np.stack([members[i]["disc"] for i in ids]),
            sign=np.stack([members[i]["sign"] for i in ids]),
            chi=np.stack([members[i]["chi"] for i in ids]),
            ledger=np.stack([members[i]["ledger"] for i in ids]),
            dims=np.stack([members[i]["dims"] for i in ids]),
            weights=weights(name, n_ckpt, every),
            checkpoints=np.arange(1, n_ckpt + 1) * every,
        )
        if name == "c1":
            payload["psi"] = np.stack([members[i]["psi"] for i in ids[:8]])
        np.savez_compressed(os.path.join(HERE, f"ref_{name}.npz"), **payload)

    # single-gate known answers (SPEC.md:291-299 examples, run through the reference API)
    kat = {}
    st = tepai.init_product_state("+++")
    tepai.apply_pauli_rotation(st, tepai.PauliString.from_label("Z0Z1", 3), math.pi / 2, tepai.TruncationPolicy(16))
    kat["zz_x0"] = tepai.expectation(st, tepai.PauliString.from_label("X0", 3))
    kat["zz_bonds"] = np.array(st.bond_dims)
    st = tepai.init_product_state("0")
    st2 = tepai.init_product_state("00")
    tepai.apply_pauli_rotation(st2, tepai.PauliString.from_label("X0", 2), math.pi, tepai.TruncationPolicy(16))
    kat["xpi_z0"] = tepai.expectation(st2, tepai.PauliString.from_label("Z0", 2))
    # ring gate on a 6-site random-ish state: exercises the swap network
    ham = tepai.build_spin_ring(6, 1.0, 11)
    st = tepai.init_product_state("0+1-0+")
    for k, t in enumerate(ham.terms):
        tepai.apply_pauli_rotation(st, t.pauli, 0.3 + 0.01 * k, tepai.TruncationPolicy(None, 1e-14))
    kat["ring6_psi"] = st.to_statevector()
    kat["ring6_dims"] = np.array(st.bond_dims)
    kat["gamma"] = np.array(tepai.gamma_coeffs(math.pi / 4, math.pi / 2))
    kat["probs"] = np.array(tepai.variant_probabilities(math.pi / 4, math.pi / 2))
    np.savez_compressed(os.path.join(HERE, "ref_kat.npz"), **kat)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
