"""C-ABI surface (library loads, exports every declared symbol — no compute
without a GPU) and the vectorised packer vs the reference lowering."""

import math
import os
import re

import numpy as np
import pytest

import paper_2604_13144_b200 as tb
from paper_2604_13144_b200 import _lib
from paper_2604_13144_b200.packing import TermTable, pack_lowered, pack_sampled
from oracle.mps_oracle import lower

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "tepai_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(tb_\w+)\s*\(", text, re.M)))


def test_library_builds_and_exports_header_symbols():
    import __graft_entry__

    __graft_entry__.build()
    lib = _lib.load()
    syms = declared_symbols()
    assert set(syms) == set(_lib.EXPORTED)
    for name in syms:
        assert hasattr(lib, name), name
    assert lib.tb_version() == 1


def decode(words):
    w = words.astype(np.int64)
    return dict(a=w & 0xFF, b=(w >> 8) & 0xFF, pa=(w >> 16) & 3, pb=(w >> 18) & 3, mr=(w >> 20) & 1,
                pi=(w >> 21) & 1, ai=w >> 22)


@pytest.mark.parametrize("n,seed", [(8, 1), (16, 3)])
def test_packed_stream_matches_reference_lowering_per_segment(n, seed):
    ham = tb.build_spin_ring(n, 1.0, 0)
    cfg = tb.PaiConfig(math.pi / 2**7, 100, 1.0)
    ckpts = np.arange(10, 101, 10)
    circ = tb.sample_circuit(ham, cfg, tb.circuit_stream(seed, 0))
    p = pack_sampled(circ, TermTable.of(ham), ckpts)
    d = decode(p.words)
    lo = 0
    for c, j in enumerate(ckpts):
        hi = int(np.searchsorted(circ.step_index, j))
        assert p.ckpt_end[c] == hi
        ga, gb, pa, pb, ang, nxt = lower(circ.slice_entries(lo, hi).operations(), n)
        sl = slice(lo, hi)
        np.testing.assert_array_equal(d["a"][sl], ga)
        np.testing.assert_array_equal(np.where(d["b"][sl] == 0xFF, -1, d["b"][sl]), gb)
        np.testing.assert_array_equal(d["pa"][sl], pa)
        np.testing.assert_array_equal(d["pb"][sl], pb)
        two = gb >= 0
        np.testing.assert_array_equal(d["mr"][sl][two], (nxt > ga)[two])
        table = np.array([cfg.delta, -cfg.delta, math.pi])
        np.testing.assert_array_equal(table[d["ai"][sl]], ang)
        n_pi = int(np.count_nonzero(circ.kinds[:hi] == 2))
        assert p.ckpt_sign[c] == 1 - 2 * (n_pi & 1)
        lo = hi


def test_pack_lowered_roundtrip():
    ham = tb.build_spin_ring(6, 1.0, 2)
    ops = [(t.pauli, 0.1 * (k + 1)) for k, t in enumerate(ham.terms)] + [(ham.terms[-1].pauli, math.pi)]
    ga, gb, pa, pb, ang, nxt = lower(ops, 6)
    words, table = pack_lowered(ga, gb, pa, pb, ang, nxt)
    d = decode(words)
    np.testing.assert_allclose(2 * np.arctan2(table[d["ai"], 1], table[d["ai"], 0]), ang, atol=1e-15)
    assert d["pi"][-1] == 1 and d["pi"][:-1].sum() == 0


def test_engine_refuses_without_device():
    """No CPU fallback: on a box without a GPU, binding a context raises."""
    try:
        import torch

        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        _lib.context(0)
