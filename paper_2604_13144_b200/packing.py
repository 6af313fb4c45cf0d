"""Vectorised packing of sampled circuits into the kernel's uint32 gate words.

Replaces the reference's per-gate Python lowering (``SampledCircuit.operations``
sampling.py:219-225 feeding ``_lower_operations`` mps.py:194-236) for the
ensemble path: the same (site a, site b, Pauli codes, angle, split look-ahead)
information is derived straight from the ``SampledCircuit`` arrays with numpy.

Look-ahead semantics: a two-site gate merges right when the *next two-site
gate of the same ``run_circuit`` call* anchors to the right of its left site
(mps.py:219-228, ``anchors`` = b-1 for non-adjacent supports, else a; the last
two-site gate of a call looks at itself).  Checkpoint segments are separate
calls (prefix semantics), so the look-ahead stops at every
checkpoint boundary.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .pauli import SYMBOL_CODE, Hamiltonian
from .sampling import PI

ONE_SITE = 0xFF
MAX_ANGLES = 1024


@dataclass(frozen=True)
class TermTable:
    """Per-term support/codes of a Hamiltonian (weight 1 or 2 terms only)."""

    a: np.ndarray
    b: np.ndarray   # -1 for one-site terms
    pa: np.ndarray
    pb: np.ndarray

    @classmethod
    def of(cls, ham: Hamiltonian) -> "TermTable":
        a, b, pa, pb = [], [], [], []
        for t in ham.terms:
            ops = t.pauli.ops
            if len(ops) == 0 or len(ops) > 2:
                raise ValueError(f"gate weight {len(ops)} is not supported")
            a.append(ops[0][0])
            pa.append(SYMBOL_CODE[ops[0][1]])
            if len(ops) == 2:
                b.append(ops[1][0])
                pb.append(SYMBOL_CODE[ops[1][1]])
            else:
                b.append(-1)
                pb.append(0)
        return cls(np.array(a, np.int64), np.array(b, np.int64), np.array(pa, np.int64), np.array(pb, np.int64))


def angle_table(angles) -> np.ndarray:
    """(n_angles, 2) table of (cos(angle/2), sin(angle/2)), as the reference
    evaluates them (``np.cos(0.5 * angle)``, _kernel.py:44-45/61-64)."""
    ang = np.asarray(angles, dtype=np.float64)
    return np.stack([np.cos(0.5 * ang), np.sin(0.5 * ang)], axis=1).copy()


def tepai_angles(delta: float) -> np.ndarray:
    """Angle table of a TE-PAI stream: index 0 = +Delta, 1 = -Delta, 2 = pi."""
    return np.array([delta, -delta, math.pi])


def encode(a, b, pa, pb, merge_right, is_pi, angle_index) -> np.ndarray:
    a = np.asarray(a, np.int64)
    b = np.asarray(b, np.int64)
    bb = np.where(b < 0, ONE_SITE, b)
    w = (a | (bb << 8) | (np.asarray(pa, np.int64) << 16) | (np.where(b < 0, 0, pb) << 18)
         | (np.asarray(merge_right, np.int64) << 20) | (np.asarray(is_pi, np.int64) << 21)
         | (np.asarray(angle_index, np.int64) << 22))
    return w.astype(np.uint32)


def merge_right_flags(a: np.ndarray, b: np.ndarray, segment_ends: np.ndarray) -> np.ndarray:
    """Look-ahead split direction for every two-site gate (see module doc)."""
    m = a.shape[0]
    anchor = np.where(b > a + 1, b - 1, a)
    nxt = anchor.copy()
    two = np.flatnonzero(b >= 0)
    if two.size:
        seg_of = np.searchsorted(segment_ends, two, side="right")
        nxt_two = anchor[two].copy()
        same = seg_of[:-1] == seg_of[1:]
        nxt_two[:-1][same] = anchor[two[1:]][same]
        nxt[two] = nxt_two
    out = np.zeros(m, np.int64)
    out[two] = (nxt[two] > a[two]).astype(np.int64)
    return out


@dataclass
class PackedSample:
    words: np.ndarray      # uint32 [nu]
    ckpt_end: np.ndarray   # int32 [C] stream position of each checkpoint
    ckpt_sign: np.ndarray  # int8 [C] sign(g) of each prefix
    nu: int


def pack_sampled(circ, table: TermTable, checkpoints: np.ndarray) -> PackedSample:
    """Pack one ``SampledCircuit`` (TE-PAI angle table ``tepai_angles``)."""
    k = circ.term_index.astype(np.int64)
    a, b = table.a[k], table.b[k]
    pa, pb = table.pa[k], table.pb[k]
    pi = circ.kinds == PI
    angle_index = np.where(pi, 2, np.where(circ.signs < 0, 1, 0))
    ends = np.searchsorted(circ.step_index, checkpoints, side="left").astype(np.int64)
    mr = merge_right_flags(a, b, ends)
    words = encode(a, b, pa, pb, mr, pi, angle_index)
    n_pi_before = np.concatenate([[0], np.cumsum(pi)])[ends]
    sign = (1 - 2 * (n_pi_before & 1)).astype(np.int8)
    return PackedSample(words, ends.astype(np.int32), sign, int(words.size))


def pack_lowered(ga, gb, pa, pb, ang, nxt):
    """Pack a reference-style lowered stream (mps.py:194-236 output) with an
    angle table of its distinct angles; returns (words, angle_cs)."""
    ang = np.asarray(ang, np.float64)
    uniq, inv = np.unique(ang, return_inverse=True)
    if uniq.size > MAX_ANGLES:
        raise ValueError("more than 1024 distinct angles in one stream")
    ga = np.asarray(ga, np.int64)
    mr = (np.asarray(nxt, np.int64) > ga).astype(np.int64)
    words = encode(ga, gb, pa, pb, mr, ang == math.pi, inv)
    return words, angle_table(uniq)


def pack_batch(samples: list[PackedSample], n_ckpt: int = 0):
    """Concatenate per-sample streams: (words, offsets[S+1], ckpt_end[S,C], ckpt_sign[S,C])."""
    if not samples:
        return (np.zeros(0, np.uint32), np.zeros(1, np.int64), np.zeros((0, n_ckpt), np.int32),
                np.zeros((0, n_ckpt), np.int8))
    offs = np.zeros(len(samples) + 1, np.int64)
    offs[1:] = np.cumsum([p.nu for p in samples])
    words = np.concatenate([p.words for p in samples]) if samples else np.zeros(0, np.uint32)
    ce = np.stack([p.ckpt_end for p in samples]).astype(np.int32)
    cs = np.stack([p.ckpt_sign for p in samples]).astype(np.int8)
    return words, offs, ce, cs
