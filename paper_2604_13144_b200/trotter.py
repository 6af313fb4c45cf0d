"""Deterministic first-order product formula (ref ``pkg/src/tepai/trotter.py:13-57``).

Used by the hybrid Trotter -> TE-PAI schedule; its continuous angles reach the
kernel through the per-run angle table of the packed gate stream.
"""

from __future__ import annotations

from dataclasses import dataclass

from .pauli import Hamiltonian, PauliString


@dataclass(frozen=True)
class TrotterCircuit:
    hamiltonian: Hamiltonian
    n_steps: int
    total_time: float
    gates: tuple[tuple[PauliString, float], ...]

    @property
    def n(self) -> int:
        return self.hamiltonian.n

    @property
    def nu(self) -> int:
        return len(self.gates)

    def operations(self):
        return iter(self.gates)


def build_trotter_circuit(ham: Hamiltonian, total_time: float, n_steps: int) -> TrotterCircuit:
    """N repetitions of the term block with angles 2 c_k T / N (ref trotter.py:48-57)."""
    if n_steps < 1:
        raise ValueError(f"n_steps must be >= 1, got {n_steps}")
    if total_time < 0:
        raise ValueError(f"negative total_time {total_time}")
    block = tuple((t.pauli, 2.0 * t.coeff * total_time / n_steps) for t in ham.terms)
    return TrotterCircuit(ham, n_steps, total_time, block * n_steps)
