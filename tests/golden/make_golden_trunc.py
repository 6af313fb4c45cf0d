"""Truncated-regime golden fixtures for the statistical parity harness
(SURVEY.md §4 test 3, §8(c) criteria (i)-(iii); VERDICT r01 "next" item 1).

Runs the UNMODIFIED reference ``tepai`` package (``/root/reference/pkg/src``,
un-jitted because its numba kernel does not compile under numba 0.65, SURVEY
§0 fact 4) on the C2 and C3 configurations for every sample id in a range, at
all 20 prefix checkpoints (SURVEY §8(a) checkpoint semantics: one
``run_circuit`` per checkpoint interval, then the reference's own
``expectation`` for every Z_j).

Each sample runs twice:
  * ``gesdd`` -- the reference exactly as shipped (``np.linalg.svd`` at
    ``_kernel.py:117`` is LAPACK zgesdd);
  * ``gesvd`` -- the same gate list with that one call swapped for LAPACK
    zgesvd (``scipy.linalg.svd(..., lapack_driver="gesvd")``), the
    ref-vs-ref spread of SURVEY §0 fact 6 / Appendix A.5.  The swap is a
    module-attribute shim in the worker process; no reference file changes.

Writes ``tests/golden/ref_c2_stat.npz`` (256 samples) and
``tests/golden/ref_c3_stat.npz`` (64 samples).  Per-sample partial results
are cached under /tmp/golden_trunc so an interrupted run resumes.

Usage:  python tests/golden/make_golden_trunc.py [--procs 7]
Cost:   ~46k CPU-s (C3 ~273 s per sample and driver un-jitted).
"""

from __future__ import annotations

import argparse
import dataclasses
import math
import os
import sys
import types

os.environ.setdefault("NUMBA_DISABLE_JIT", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CACHE = os.environ.get("GOLDEN_TRUNC_CACHE", "/tmp/golden_trunc")
DELTA = math.pi / 2**7
CONFIGS = {
    # name: (n, ham_seed, circ_seed, n_steps, T, chi, n_samples)
    "c2": (16, 2, 3, 200, 2.0, 32, 256),
    "c3": (32, 4, 5, 200, 2.0, 64, 64),
}
N_CKPT, EVERY = 20, 10


def _select_driver(driver: str):
    """Point the reference kernel's ``np`` at numpy itself (gesdd, as shipped)
    or at a shim whose ``linalg.svd`` is zgesvd.  Called for EVERY job: pool
    workers are reused, so the choice must never leak into the next job."""
    import scipy.linalg
    from tepai import _kernel

    if driver == "gesdd":
        _kernel.np = np
        return

    if driver == "gesdd_t":
        # zgesdd on the conjugate transpose: the same LAPACK driver, but an
        # independent bidiagonalisation (zgesdd and zgesvd on the SAME matrix
        # share zgebrd), i.e. a twin that differs from the shipped reference the
        # way an independent SVD algorithm of the same accuracy class does
        def svd(a, full_matrices=True):
            u, sv, vh = np.linalg.svd(np.ascontiguousarray(a.conj().T), full_matrices=full_matrices)
            return np.ascontiguousarray(vh.conj().T), sv, np.ascontiguousarray(u.conj().T)
    else:
        def svd(a, full_matrices=True):
            return scipy.linalg.svd(a, full_matrices=full_matrices, lapack_driver="gesvd", check_finite=False)

    shim = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np) if not k.startswith("__")})
    shim.linalg = types.SimpleNamespace(svd=svd, qr=np.linalg.qr)
    _kernel.np = shim


def run_member(args):
    name, sid, driver = args
    path = os.path.join(CACHE, f"{name}_{driver}_{sid}.npz")
    if os.path.exists(path):
        return path
    import tepai
    from tepai import _kernel
    from tepai import rng as trng
    _select_driver(driver)
    assert (_kernel.np is np) == (driver == "gesdd")
    n, hs, cs, steps, T, chi, _ = CONFIGS[name]
    ham = tepai.build_spin_ring(n, 1.0, hs)
    circ = tepai.sample_circuit(ham, tepai.PaiConfig(DELTA, steps, T), trng.circuit_stream(cs, sid), sample_id=sid)
    state = tepai.init_product_state("01" * (n // 2))
    policy = tepai.TruncationPolicy(chi_cut=chi, svalue_floor=1e-12)
    ledger = tepai.CostLedger()
    zs = [tepai.PauliString.single(n, q, "Z") for q in range(n)]
    vals = np.zeros((N_CKPT, n))
    disc = np.zeros(N_CKPT)
    sign = np.zeros(N_CKPT, np.int64)
    lo = 0
    for ci in range(N_CKPT):
        j = (ci + 1) * EVERY
        hi = int(np.searchsorted(circ.step_index, j, side="left"))
        seg = dataclasses.replace(circ, term_index=circ.term_index[lo:hi], step_index=circ.step_index[lo:hi],
                                  kinds=circ.kinds[lo:hi], signs=circ.signs[lo:hi])
        tepai.run_circuit(state, seg, policy, ledger)
        lo = hi
        vals[ci] = [tepai.expectation(state, z) for z in zs]
        disc[ci] = tepai.discarded_weight(state)
        sign[ci] = 1 - 2 * (int(np.count_nonzero(circ.kinds[:hi] == 2)) & 1)
    os.makedirs(CACHE, exist_ok=True)
    tmp = path + ".part.npz"
    np.savez(tmp, vals=vals, disc=disc, sign=sign,
             ledger=np.array([ledger.gate_count, ledger.sum_chi_cubed, ledger.chi_max], np.float64))
    os.replace(tmp, path)
    return path


def purge_leaked(names):
    """Drop cached gesdd results that are bit-identical to their gesvd twin at
    the last checkpoint (made by an earlier version of this script whose
    workers kept the zgesvd shim installed); they are recomputed."""
    for nm in names:
        for i in range(CONFIGS[nm][6]):
            a = os.path.join(CACHE, f"{nm}_gesdd_{i}.npz")
            b = os.path.join(CACHE, f"{nm}_gesvd_{i}.npz")
            if os.path.exists(a) and os.path.exists(b):
                va, vb = np.load(a)["vals"], np.load(b)["vals"]
                if np.array_equal(va[-1], vb[-1]):
                    os.remove(a)


def assemble(name):
    import tepai
    n, hs, cs, steps, T, chi, count = CONFIGS[name]
    ham = tepai.build_spin_ring(n, 1.0, hs)
    weights = np.array([tepai.sampling.circuit_weight_norm(
        ham, tepai.PaiConfig(DELTA, (c + 1) * EVERY, (c + 1) * EVERY * T / steps)) for c in range(N_CKPT)])
    out = dict(sample_ids=np.arange(count), weights=weights, checkpoints=np.arange(1, N_CKPT + 1) * EVERY)
    for driver in ("gesdd", "gesvd"):
        rows = [np.load(os.path.join(CACHE, f"{name}_{driver}_{i}.npz")) for i in range(count)]
        out[f"vals_{driver}"] = np.stack([r["vals"] for r in rows])
        out[f"disc_{driver}"] = np.stack([r["disc"] for r in rows])
        out[f"ledger_{driver}"] = np.stack([r["ledger"] for r in rows])
        if driver == "gesdd":
            out["sign"] = np.stack([r["sign"] for r in rows])
    np.savez_compressed(os.path.join(HERE, f"ref_{name}_stat.npz"), **out)


def main():
    from multiprocessing import Pool
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--only", choices=sorted(CONFIGS), default=None)
    ap.add_argument("--third-twin", type=int, default=0, metavar="N",
                    help="only run the first N samples of --only with zgesdd on the conjugate transpose and write "
                         "ref_<config>_stat_twinT.npz (the spread an independent bidiagonalisation gives)")
    a = ap.parse_args()
    if a.third_twin:
        nm = a.only or "c3"
        jobs = [(nm, i, "gesdd_t") for i in range(a.third_twin)]
        with Pool(a.procs) as pool:
            for k, p in enumerate(pool.imap_unordered(run_member, jobs, chunksize=1)):
                print(f"[{k + 1}/{len(jobs)}] {os.path.basename(p)}", flush=True)
        rows = [np.load(os.path.join(CACHE, f"{nm}_gesdd_t_{i}.npz")) for i in range(a.third_twin)]
        np.savez_compressed(os.path.join(HERE, f"ref_{nm}_stat_twinT.npz"), sample_ids=np.arange(a.third_twin),
                            vals_gesdd_t=np.stack([r["vals"] for r in rows]),
                            disc_gesdd_t=np.stack([r["disc"] for r in rows]))
        print("written:", f"ref_{nm}_stat_twinT.npz")
        return
    names = [a.only] if a.only else ["c2", "c3"]
    purge_leaked(names)
    jobs = [(nm, i, d) for nm in names for i in range(CONFIGS[nm][6]) for d in ("gesdd", "gesvd")]
    with Pool(a.procs) as pool:
        for k, p in enumerate(pool.imap_unordered(run_member, jobs, chunksize=1)):
            print(f"[{k + 1}/{len(jobs)}] {os.path.basename(p)}", flush=True)
    purge_leaked(names)
    missing = [j for j in jobs if not os.path.exists(os.path.join(CACHE, f"{j[0]}_{j[2]}_{j[1]}.npz"))]
    if missing:
        raise SystemExit(f"{len(missing)} results were purged as driver leaks; run the script again")
    for nm in names:
        assemble(nm)
    print("written:", [f"ref_{nm}_stat.npz" for nm in names])


if __name__ == "__main__":
    main()
