"""Golden fixture for the hybrid Trotter -> TE-PAI schedule (config 5 at desk
scale), produced with the UNMODIFIED reference (un-jitted, see make_golden.py):
first-order Trotter evolution of the Neel state on a 6-site ring to t0, then
TE-PAI continuations (prefix checkpoints) of 16 samples from that MPS.

Usage: python tests/golden/make_golden_hybrid.py     Writes: tests/golden/ref_hybrid_n6.npz
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
N, HSEED, CSEED = 6, 8, 9
T0, TROTTER_STEPS = 0.6, 30
DELTA, STEPS, T = math.pi / 2**6, 20, 0.4
CKPT = [5, 10, 15, 20]


def main():
    ham = tepai.build_spin_ring(N, 1.0, HSEED)
    policy = tepai.TruncationPolicy(chi_cut=8, svalue_floor=1e-12)
    st0 = tepai.init_product_state("01" * (N // 2))
    tepai.run_circuit(st0, tepai.build_trotter_circuit(ham, T0, TROTTER_STEPS), policy)
    z0 = [tepai.expectation(st0, tepai.PauliString.single(N, q, "Z")) for q in range(N)]
    snap = tepai.mps.snapshot_to_bytes(st0)
    cfg = tepai.PaiConfig(DELTA, STEPS, T)
    vals = np.zeros((16, len(CKPT), N))
    sign = np.zeros((16, len(CKPT)), np.int64)
    for i in range(16):
        circ = tepai.sample_circuit(ham, cfg, trng.circuit_stream(CSEED, i), sample_id=i)
        st = tepai.mps.snapshot_from_bytes(snap)
        lo = 0
        for c, j in enumerate(CKPT):
            hi = int(np.searchsorted(circ.step_index, j))
            seg = dataclasses.replace(circ, term_index=circ.term_index[lo:hi], step_index=circ.step_index[lo:hi],
                                      kinds=circ.kinds[lo:hi], signs=circ.signs[lo:hi])
            tepai.run_circuit(st, seg, policy)
            lo = hi
            vals[i, c] = [tepai.expectation(st, tepai.PauliString.single(N, q, "Z")) for q in range(N)]
            sign[i, c] = 1 - 2 * (int(np.count_nonzero(circ.kinds[:hi] == 2)) & 1)
    np.savez_compressed(os.path.join(HERE, "ref_hybrid_n6.npz"), z_t0=np.array(z0), vals=vals, sign=sign,
                        psi_t0=st0.to_statevector(), dims_t0=np.array(st0.dims), checkpoints=np.array(CKPT))
    print("written", vals.shape)


if __name__ == "__main__":
    main()
