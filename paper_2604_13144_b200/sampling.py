"""TE-PAI quasiprobability weights and the seeded circuit-variant sampler.

Host-side restatement of ``pkg/src/tepai/sampling.py``.  The draw sequence
(which generator calls happen, in which order, with which shapes) follows the
reference line by line so that the sampled gate lists are bit-identical:

* ``gamma_coeffs`` / ``variant_probabilities`` — ref sampling.py:96-120
* per-slot probability table — ref sampling.py:123-135
* ``circuit_weight_norm`` (finite-N overhead ||g||_1) — ref sampling.py:138-153
* ``sample_circuit`` grid / runs methods — ref sampling.py:244-321
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .pauli import Hamiltonian

IDENTITY, DELTA, PI = 0, 1, 2
GRID_METHOD_CUTOFF = 4096  # ref sampling.py:241
DELTA_MIN_GATES = 2.0 * math.atan(1.0 / math.sqrt(2.0))


@dataclass(frozen=True)
class PaiConfig:
    """Interpolation angle, step count, time span, mode (ref sampling.py:55-84)."""

    delta: float
    n_steps: int
    total_time: float
    mode: str = "unbiased"

    def __post_init__(self):
        if not 0.0 < self.delta <= math.pi:
            raise ValueError(f"delta must lie in (0, pi], got {self.delta}")
        if self.n_steps < 1:
            raise ValueError(f"n_steps must be >= 1, got {self.n_steps}")
        if self.total_time < 0:
            raise ValueError(f"negative total_time {self.total_time}")
        if self.mode not in ("unbiased", "no_pi"):
            raise ValueError(f"unknown mode {self.mode!r}")

    def angles(self, ham: Hamiltonian) -> np.ndarray:
        """theta_k = 2 c_k T / N, evaluated in the reference's operation order."""
        return 2.0 * ham.coefficients() * self.total_time / self.n_steps

    def validate_against(self, ham: Hamiltonian) -> None:
        worst = float(np.max(np.abs(self.angles(ham)), initial=0.0))
        if worst > self.delta * (1.0 + 1e-12):
            raise ValueError(
                f"delta={self.delta} smaller than the largest rotation angle {worst}; "
                "increase n_steps or delta"
            )


def _clip_theta(theta: float, delta: float) -> float:
    if not 0.0 < delta <= math.pi:
        raise ValueError(f"delta must lie in (0, pi], got {delta}")
    t = abs(theta)
    if t > delta * (1.0 + 1e-12):
        raise ValueError(f"|theta|={t} exceeds delta={delta}")
    return min(t, delta)


def gamma_coeffs(theta: float, delta: float) -> tuple[float, float, float]:
    """(gamma1, gamma2, gamma3) at |theta| (ref sampling.py:96-107)."""
    t = _clip_theta(theta, delta)
    gap = math.sin(0.5 * (delta - t))
    return (
        math.cos(0.5 * t) * gap / math.sin(0.5 * delta),
        math.sin(t) / math.sin(delta),
        -math.sin(0.5 * t) * gap / math.cos(0.5 * delta),
    )


def gamma_l1_norm(theta: float, delta: float) -> float:
    """|g1|+|g2|+|g3| in cancellation-free form (ref sampling.py:110-113)."""
    t = _clip_theta(theta, delta)
    return 1.0 + 2.0 * math.sin(0.5 * t) * math.sin(0.5 * (delta - t)) / math.cos(0.5 * delta)


def variant_probabilities(theta: float, delta: float) -> tuple[float, float, float]:
    """p_l = |gamma_l| / sum |gamma| (ref sampling.py:116-120)."""
    g = [abs(x) for x in gamma_coeffs(theta, delta)]
    norm = g[0] + g[1] + g[2]
    return g[0] / norm, g[1] / norm, g[2] / norm


def slot_probabilities(ham: Hamiltonian, cfg: PaiConfig) -> np.ndarray:
    """(L, 3) per-term variant probabilities (ref sampling.py:123-135)."""
    thetas = np.abs(cfg.angles(ham))
    probs = np.empty((len(thetas), 3))
    if cfg.mode == "no_pi":
        lam = thetas / cfg.delta
        probs[:, 0], probs[:, 1], probs[:, 2] = 1.0 - lam, lam, 0.0
    else:
        for k, t in enumerate(thetas):
            probs[k] = variant_probabilities(t, cfg.delta)
    return probs


def circuit_weight_norm(ham: Hamiltonian, cfg: PaiConfig) -> float:
    """||g||_1 = prod over N*L slots of the per-gate norm (ref sampling.py:138-153)."""
    cfg.validate_against(ham)
    if cfg.mode == "no_pi":
        return 1.0
    acc = 0.0
    for t in np.abs(cfg.angles(ham)):
        tt = min(float(t), cfg.delta)
        acc += math.log1p(2.0 * math.sin(0.5 * tt) * math.sin(0.5 * (cfg.delta - tt)) / math.cos(0.5 * cfg.delta))
    return math.exp(cfg.n_steps * acc)


def expected_gate_count_inf(delta: float, c_norm: float, total_time: float) -> float:
    """csc(D)(3 - cos D)|c|_1 T (ref sampling.py:156-162)."""
    if not 0.0 < delta <= math.pi:
        raise ValueError(f"delta must lie in (0, pi], got {delta}")
    if total_time < 0:
        raise ValueError(f"negative total_time {total_time}")
    return (3.0 - math.cos(delta)) / math.sin(delta) * c_norm * total_time


def overhead_norm_inf(delta: float, c_norm: float, total_time: float) -> float:
    """exp[2 tan(D/2)|c|_1 T] (ref sampling.py:165-171)."""
    if not 0.0 < delta < math.pi:
        raise ValueError(f"delta must lie in (0, pi), got {delta}")
    if total_time < 0:
        raise ValueError(f"negative total_time {total_time}")
    return math.exp(2.0 * math.tan(0.5 * delta) * c_norm * total_time)


@dataclass(frozen=True)
class SampledCircuit:
    """Columnar circuit variant, entries in (step, term) order (ref sampling.py:185-225)."""

    hamiltonian: Hamiltonian
    config: PaiConfig
    term_index: np.ndarray
    step_index: np.ndarray
    kinds: np.ndarray
    signs: np.ndarray
    overall_sign: int
    weight_norm: float
    sample_id: int = 0

    @property
    def nu(self) -> int:
        return len(self.term_index)

    @property
    def n(self) -> int:
        return self.hamiltonian.n

    def operations(self):
        """(PauliString, angle) pairs: pi for PI draws, sign*Delta otherwise."""
        terms = self.hamiltonian.terms
        d = self.config.delta
        for k, kind, s in zip(self.term_index, self.kinds, self.signs):
            yield terms[k].pauli, (math.pi if kind == PI else float(s) * d)

    def prefix(self, n_steps: int) -> "SampledCircuit":
        """Entries with step_index < n_steps (used for checkpoint segments)."""
        cut = int(np.searchsorted(self.step_index, n_steps, side="left"))
        return self.slice_entries(0, cut)

    def slice_entries(self, lo: int, hi: int) -> "SampledCircuit":
        return SampledCircuit(
            self.hamiltonian, self.config, self.term_index[lo:hi], self.step_index[lo:hi],
            self.kinds[lo:hi], self.signs[lo:hi], self.overall_sign, self.weight_norm, self.sample_id,
        )


def _sorted_subset(rng: np.random.Generator, n: int, m: int) -> np.ndarray:
    """Uniform sorted m-subset of range(n) (ref sampling.py:228-237)."""
    if 4 * m * m <= n:
        while True:
            picks = np.unique(rng.integers(0, n, size=m))
            if picks.size == m:
                return picks
    return np.sort(rng.permutation(n)[:m])


def _draw_grid(rng, probs, n_steps):
    u = rng.random((n_steps, probs.shape[0]))
    lo = probs[:, 0]
    hi = probs[:, 0] + probs[:, 1]
    variant = np.where(u < lo, IDENTITY, np.where(u < hi, DELTA, PI))
    jj, kk = np.nonzero(variant)
    return kk.astype(np.int32), jj.astype(np.int32), variant[jj, kk].astype(np.int8)


def _draw_runs(rng, probs, n_steps):
    ks, js, vs = [], [], []
    for k in range(probs.shape[0]):
        q = probs[k, 1] + probs[k, 2]
        if q <= 0.0:
            continue
        m = int(rng.binomial(n_steps, q))
        if m == 0:
            continue
        steps = _sorted_subset(rng, n_steps, m)
        if probs[k, 2] == 0.0:
            kind = np.full(m, DELTA, dtype=np.int8)
        else:
            kind = np.where(rng.random(m) < probs[k, 1] / q, DELTA, PI).astype(np.int8)
        ks.append(np.full(m, k, dtype=np.int32))
        js.append(steps.astype(np.int32))
        vs.append(kind)
    if not ks:
        return np.zeros(0, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int8)
    kk, jj, vv = np.concatenate(ks), np.concatenate(js), np.concatenate(vs)
    order = np.lexsort((kk, jj))
    return kk[order], jj[order], vv[order]


def sample_circuit(ham: Hamiltonian, cfg: PaiConfig, rng: np.random.Generator,
                   sample_id: int = 0, method: str = "auto") -> SampledCircuit:
    """Draw one circuit variant over the N x L slot grid (ref sampling.py:244-321)."""
    cfg.validate_against(ham)
    probs = slot_probabilities(ham, cfg)
    L, N = ham.num_terms, cfg.n_steps
    term_signs = np.sign(ham.coefficients()).astype(np.int8) if L else np.zeros(0, np.int8)
    if method == "auto":
        method = "runs" if N * L > GRID_METHOD_CUTOFF else "grid"
    if method == "grid":
        if L == 0:
            kk = jj = np.zeros(0, np.int32)
            vv = np.zeros(0, np.int8)
        else:
            kk, jj, vv = _draw_grid(rng, probs, N)
    elif method == "runs":
        kk, jj, vv = _draw_runs(rng, probs, N)
    else:
        raise ValueError(f"unknown sampling method {method!r}")
    if len(kk):
        signs = np.where(vv == DELTA, term_signs[kk], 1).astype(np.int8)
    else:
        signs = np.ones(0, np.int8)
    n_pi = int(np.count_nonzero(vv == PI))
    return SampledCircuit(ham, cfg, kk, jj, vv, signs, 1 - 2 * (n_pi & 1),
                          circuit_weight_norm(ham, cfg), sample_id)
