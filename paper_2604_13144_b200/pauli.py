"""Pauli strings and the disordered spin-ring Hamiltonian (host side).

Restates the parts of ``pkg/src/tepai/pauli.py`` that the ensemble path
consumes: ``PauliString`` (ref :36-103), ``HamTerm``/``Hamiltonian``
(ref :130-167) and ``build_spin_ring`` (ref :170-207).  Term order and the
disorder draw are reproduced exactly, because the sampler indexes terms by
position and the gate lists must be bit-identical to the reference's.
"""

from __future__ import annotations

import math
import re
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from .rng import disorder_stream

SYMBOL_CODE = {"X": 1, "Y": 2, "Z": 3}
_LABEL_TOKEN = re.compile(r"([XYZ])(\d+)")
_MATS = {
    "I": np.eye(2, dtype=complex),
    "X": np.array([[0, 1], [1, 0]], dtype=complex),
    "Y": np.array([[0, -1j], [1j, 0]], dtype=complex),
    "Z": np.array([[1, 0], [0, -1]], dtype=complex),
}


@dataclass(frozen=True)
class PauliString:
    """Non-identity support of an ``n``-qubit Pauli product, sorted by site
    (ref pauli.py:36-59)."""

    n: int
    ops: tuple[tuple[int, str], ...] = ()

    def __post_init__(self):
        if self.n < 1:
            raise ValueError(f"qubit count must be positive, got {self.n}")
        sites = [s for s, _ in self.ops]
        for s, sym in self.ops:
            if not 0 <= s < self.n:
                raise ValueError(f"support site {s} outside [0, {self.n})")
            if sym not in SYMBOL_CODE:
                raise ValueError(f"invalid Pauli symbol {sym!r}")
        if len(set(sites)) != len(sites):
            raise ValueError("duplicate site in Pauli support")
        object.__setattr__(self, "ops", tuple(sorted(self.ops)))

    @classmethod
    def from_label(cls, label: str, n: int) -> "PauliString":
        label = label.strip()
        if label in ("", "I"):
            return cls(n)
        toks = _LABEL_TOKEN.findall(label)
        if "".join(f"{s}{q}" for s, q in toks) != label:
            raise ValueError(f"malformed Pauli label {label!r}")
        return cls(n, tuple((int(q), s) for s, q in toks))

    @classmethod
    def single(cls, n: int, site: int, sym: str) -> "PauliString":
        return cls(n, ((site, sym),))

    @property
    def weight(self) -> int:
        return len(self.ops)

    @property
    def support(self) -> tuple[int, ...]:
        return tuple(s for s, _ in self.ops)

    def symbol_at(self, site: int) -> str:
        return dict(self.ops).get(site, "I")

    def label(self) -> str:
        return "".join(f"{sym}{s}" for s, sym in self.ops) or "I"

    __str__ = label

    def matrix(self) -> np.ndarray:
        """Dense matrix, site 0 most significant (test helper, small n only)."""
        out = np.ones((1, 1), dtype=complex)
        for s in range(self.n):
            out = np.kron(out, _MATS[self.symbol_at(s)])
        return out


@dataclass(frozen=True)
class HamTerm:
    """Weighted Pauli term; zero/non-finite weights rejected (ref pauli.py:130-141)."""

    coeff: float
    pauli: PauliString

    def __post_init__(self):
        if not math.isfinite(self.coeff):
            raise ValueError(f"non-finite coefficient {self.coeff}")
        if self.coeff == 0.0:
            raise ValueError("zero-coefficient terms must be dropped at construction")


@dataclass(frozen=True)
class Hamiltonian:
    """Ordered term list; the order fixes the product formula (ref pauli.py:144-167)."""

    n: int
    terms: tuple[HamTerm, ...]
    coupling: float = 0.0
    seed: int | None = None

    def __post_init__(self):
        if any(t.pauli.n != self.n for t in self.terms):
            raise ValueError("term qubit count differs from Hamiltonian")

    @property
    def num_terms(self) -> int:
        return len(self.terms)

    def coefficients(self) -> np.ndarray:
        return np.array([t.coeff for t in self.terms])


def build_spin_ring(n: int, coupling: float, omega: Sequence[float] | int) -> Hamiltonian:
    """Periodic disordered Heisenberg ring (ref pauli.py:170-207).

    Terms: ``Z_k`` fields for k = 0..n-1 (dropped when the field is exactly
    zero), then for every bond b = 0..n-1 the couplings X_bX_{b+1},
    Y_bY_{b+1}, Z_bZ_{b+1}; the wrap bond is stored with sorted support
    (0, n-1) so it is the only non-adjacent pair.  An integer ``omega`` is a
    seed: fields ~ U[-1, 1] from ``disorder_stream(seed)``.
    """
    if n < 3:
        raise ValueError(f"ring needs n >= 3, got {n}")
    if not math.isfinite(coupling):
        raise ValueError("non-finite coupling")
    seed = None
    if isinstance(omega, (int, np.integer)):
        seed = int(omega)
        fields = disorder_stream(seed).uniform(-1.0, 1.0, size=n)
    else:
        fields = np.asarray(omega, dtype=float)
        if fields.shape != (n,):
            raise ValueError(f"omega must have length {n}, got shape {fields.shape}")
        if not np.all(np.isfinite(fields)):
            raise ValueError("non-finite omega values")
    terms = [HamTerm(float(fields[k]), PauliString.single(n, k, "Z")) for k in range(n) if fields[k] != 0.0]
    if coupling != 0.0:
        for b in range(n):
            pair = (b, (b + 1) % n)
            terms.extend(HamTerm(float(coupling), PauliString(n, tuple((q, sym) for q in pair))) for sym in "XYZ")
    return Hamiltonian(n, tuple(terms), coupling=float(coupling), seed=seed)


def coeff_l1_norm(ham: Hamiltonian) -> float:
    """Sum of |c_k| (ref pauli.py:210-212)."""
    return float(sum(abs(t.coeff) for t in ham.terms))


def build_tfim_ring(n: int, field: float, seed: int, j_range=(0.5, 1.5), h_range=(-1.0, 1.0)) -> Hamiltonian:
    """Periodic disordered transverse-field Ising ring (BASELINE config 4):
    H = sum_j J_j Z_j Z_{j+1} + g sum_j X_j + sum_j h_j Z_j.

    The reference ships only the generic ``Hamiltonian``/``HamTerm`` types
    (ref pauli.py:130-167) and no TFIM builder, so this module fixes the two
    conventions the config leaves open, mirroring ``build_spin_ring``
    (ref pauli.py:170-207):
    - draw order: ``J = U[j_range]`` for bonds 0..n-1, then ``h = U[h_range]``
      for sites 0..n-1, both from ``disorder_stream(seed)``;
    - term order: the Z fields h_k Z_k by site, then the X fields g X_k by site,
      then the couplings J_b Z_b Z_{b+1} by bond, the wrap bond stored sorted
      as Z_0 Z_{n-1} (the only non-adjacent pair).
    Zero coefficients are dropped as in the reference builder.
    """
    if n < 3:
        raise ValueError(f"ring needs n >= 3, got {n}")
    if not math.isfinite(field):
        raise ValueError("non-finite transverse field")
    rng = disorder_stream(int(seed))
    couplings = rng.uniform(j_range[0], j_range[1], size=n)
    fields = rng.uniform(h_range[0], h_range[1], size=n)
    terms = [HamTerm(float(fields[k]), PauliString.single(n, k, "Z")) for k in range(n) if fields[k] != 0.0]
    if field != 0.0:
        terms.extend(HamTerm(float(field), PauliString.single(n, k, "X")) for k in range(n))
    for b in range(n):
        if couplings[b] != 0.0:
            pair = (b, (b + 1) % n)
            terms.append(HamTerm(float(couplings[b]), PauliString(n, tuple((q, "Z") for q in pair))))
    return Hamiltonian(n, tuple(terms), coupling=0.0, seed=int(seed))


def min_trotter_steps(ham: Hamiltonian, delta: float, total_time: float) -> int:
    """Smallest step count N with max_k |2 c_k T / N| <= delta, i.e. the first
    N that ``PaiConfig.validate_against`` (ref sampling.py:64-84) accepts."""
    cmax = max(abs(t.coeff) for t in ham.terms)
    steps = max(1, math.ceil(2.0 * cmax * total_time / delta))
    while 2.0 * cmax * total_time / steps > delta * (1.0 + 1e-12):
        steps += 1
    while steps > 1 and 2.0 * cmax * total_time / (steps - 1) <= delta * (1.0 + 1e-12):
        steps -= 1
    return steps
