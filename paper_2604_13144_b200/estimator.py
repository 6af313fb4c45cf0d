"""Signed, Gamma-weighted ensemble estimator (the reference
package has no code for it).

Per sample l and time t:  v_l = sign(g_l) <O>_l  (|v| <= 1),  o_l = ||g||_1 v_l.
mean = (1/Ns) sum o_l;  Var[v] and Var[o] with the unbiased (Ns - 1)
denominator;  Var[o] = ||g||_1^2 Var[v] exactly when ||g||_1 is common to the
ensemble (checked to 1e-12).

The device accumulates sum v and sum v^2 per (checkpoint, site) in 2^-40
fixed point (int64), so partial sums from any number of CTAs, GPUs or ranks
combine associatively and the statistics are bit-identical for every worker
count.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

FIX_BITS = 40
FIX = float(2**FIX_BITS)
TABLE_COLUMNS = ("t", "estimate", "std_error", "var_o", "var_v", "g_norm", "mean_nu", "mean_cost", "chi_max")


@dataclass(frozen=True)
class SampleRecord:
    """One ensemble member's contribution at one time."""

    sample_id: int
    sign: int
    weight_norm: float
    value: float          # raw <O> without the sign
    nu: int = 0
    cost: float = 0.0
    config: tuple = ()

    @property
    def v(self) -> float:
        return self.sign * self.value

    @property
    def o(self) -> float:
        return self.weight_norm * self.v


@dataclass
class EnsembleResult:
    n_samples: int
    mean: float
    var_o: float
    var_v: float
    g_norm: float
    std_error: float
    mean_nu: float = 0.0
    mean_cost: float = 0.0
    chi_max: int = 0
    records: list = field(default_factory=list)


def _finish(ns: int, sum_v: float, sum_v2: float, g: float, **extra) -> EnsembleResult:
    mean_v = sum_v / ns
    var_v = (sum_v2 - ns * mean_v * mean_v) / (ns - 1) if ns > 1 else 0.0
    var_v = max(var_v, 0.0)
    var_o = g * g * var_v
    return EnsembleResult(ns, g * mean_v, var_o, var_v, g, math.sqrt(var_o / ns), **extra)


def aggregate(records) -> EnsembleResult:
    """SPEC.md:419-427 aggregate over per-sample records."""
    recs = list(records)
    if not recs:
        raise ValueError("aggregate needs at least one sample")
    cfgs = {r.config for r in recs}
    if len(cfgs) > 1:
        raise ValueError("samples come from mixed configurations")
    g = recs[0].weight_norm
    if any(r.weight_norm != g for r in recs):
        raise ValueError("weight_norm differs across samples (mixed Delta, N, T or mode)")
    v = np.array([r.v for r in recs])
    o = g * v
    ns = len(recs)
    res = EnsembleResult(
        n_samples=ns,
        mean=float(o.mean()),
        var_o=float(o.var(ddof=1)) if ns > 1 else 0.0,
        var_v=float(v.var(ddof=1)) if ns > 1 else 0.0,
        g_norm=g,
        std_error=0.0,
        mean_nu=float(np.mean([r.nu for r in recs])),
        mean_cost=float(np.mean([r.cost for r in recs])),
        records=recs,
    )
    res.std_error = math.sqrt(res.var_o / ns)
    if abs(res.var_o - g * g * res.var_v) > 1e-12 * max(1.0, res.var_o):
        raise AssertionError("scaling identity Var[o] = ||g||^2 Var[v] violated")
    return res


def aggregate_fixed(sum_v: np.ndarray, sum_v2: np.ndarray, n_samples, g_norm: np.ndarray):
    """Statistics from the device's fixed-point sums: arrays [C, O] of int64,
    g_norm [C]; ``n_samples`` is one count or one per checkpoint row [C] (rows
    can differ when the engine left a non-converged sample out).  Returns dict
    of float arrays (mean, std_error, var_o, var_v)."""
    ns = np.asarray(n_samples, dtype=np.int64)
    if ns.size == 0 or int(ns.min()) < 1:
        raise ValueError("aggregate needs at least one sample")
    sv = np.asarray(sum_v, dtype=np.int64).astype(np.float64) / FIX
    sv2 = np.asarray(sum_v2, dtype=np.int64).astype(np.float64) / FIX
    g = np.asarray(g_norm, dtype=np.float64).reshape(-1, 1)
    n = ns.astype(np.float64).reshape(-1, 1) if ns.ndim else float(ns)
    mean_v = sv / n
    var_v = np.where(n > 1, np.maximum((sv2 - n * mean_v * mean_v) / np.maximum(n - 1, 1), 0.0), 0.0)
    var_o = g * g * var_v
    return {"estimate": g * mean_v, "std_error": np.sqrt(var_o / n), "var_o": var_o, "var_v": var_v,
            "mean_v": mean_v}


def quantize(v) -> np.ndarray:
    """Host replica of the device rounding (llrint(v * 2^40))."""
    return np.rint(np.asarray(v, dtype=np.float64) * FIX).astype(np.int64)


def results_table(times, stats: dict, g_norm, site: int, mean_nu=0.0, mean_cost=0.0, chi_max=0) -> str:
    """Comma-separated results table (SPEC.md:463 columns), one row per time."""
    lines = [",".join(TABLE_COLUMNS)]
    for c, t in enumerate(times):
        lines.append(",".join(repr(float(x)) if not isinstance(x, int) else str(x) for x in (
            float(t), float(stats["estimate"][c, site]), float(stats["std_error"][c, site]),
            float(stats["var_o"][c, site]), float(stats["var_v"][c, site]), float(g_norm[c]),
            float(mean_nu), float(mean_cost), int(chi_max))))
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# Signed mixture (PAPER §II.C): rho(t) is the
# Gamma-weighted signed average of the retained per-sample states, so any
# observable is extracted in one pass over them, without re-simulation.
# ---------------------------------------------------------------------------
@dataclass
class SignedMixture:
    """(sign, MPS snapshot) pairs with the shared scale ||g||_1 / N_s."""

    signs: np.ndarray        # int [S], sign(g_l) of each sample at the mixture's time
    weight_norm: float       # ||g||_1 at that time (common to the ensemble)
    states: np.ndarray       # complex128 [S, n, cap, 2, cap]
    dims: np.ndarray         # int [S, n+1]
    sample_ids: np.ndarray | None = None

    @property
    def n_samples(self) -> int:
        return int(self.signs.size)

    @property
    def scale(self) -> float:
        return self.weight_norm / self.n_samples


def mixture_from_run(run) -> SignedMixture:
    """The signed mixture of an ``EnsembleRun`` made with ``retain_states=True``:
    the final states, each sample's sign at the last checkpoint, and the last
    checkpoint's ||g||_1."""
    if run.states is None:
        raise ValueError("snapshots not retained: run the ensemble with retain_states=True")
    if run.signs is None or run.signs.shape[1] == 0:
        raise ValueError("the run has no checkpoint to attach the mixture to")
    return SignedMixture(np.asarray(run.signs[:, -1], dtype=np.int64), float(run.weights[-1]), run.states,
                         run.state_dims.astype(np.int64), run.sample_ids)


def _codes(pauli, n: int) -> np.ndarray:
    sym = {"X": 1, "Y": 2, "Z": 3}
    c = np.zeros(n, np.int32)
    for site, s in pauli.ops:
        c[site] = sym[s]
    return c


def per_sample_expectations(mixture: SignedMixture, observables, device: int = 0) -> np.ndarray:
    """<psi_l|P_o|psi_l> for every retained state and observable, [S, O]
    (one batched engine call, ``tb_expectation_batch``)."""
    import ctypes  # noqa: F401  (ctypes pointers through _lib)

    from . import _lib

    S, n, cap = mixture.states.shape[0], mixture.states.shape[1], mixture.states.shape[2]
    obs = list(observables)
    for o in obs:
        if o.n != n:
            raise ValueError("observable qubit count differs from the mixture's states")
    codes = np.ascontiguousarray(np.stack([_codes(o, n) for o in obs]) if obs else np.zeros((0, n), np.int32))
    out = np.zeros((S, len(obs)))
    bufs = np.ascontiguousarray(mixture.states)
    dims = np.ascontiguousarray(mixture.dims, dtype=np.int64)
    ctx = _lib.context(device)
    _lib.check(_lib.load().tb_expectation_batch(ctx, bufs.ctypes.data, S, n, cap, dims.ctypes.data, codes.ctypes.data,
                                                len(obs), out.ctypes.data), ctx)
    return out


def evaluate_observables(mixture: SignedMixture, observables, device: int = 0) -> list:
    """Tr[O rho(t)] = (||g||_1 / N_s) sum_l sign_l <psi_l|O|psi_l> for each
    observable: equal to ``aggregate`` of that observable
    computed sample-wise."""
    if mixture.states is None:
        raise ValueError("snapshots not retained")
    vals = per_sample_expectations(mixture, observables, device)
    return [float(x) for x in mixture.scale * (mixture.signs[:, None] * vals).sum(axis=0)]


def variance_vs_bound_trace(times, stats: dict, g_norm, site: int = 0, n_samples=None, slack: float | None = None):
    """Rows (t, Var[o], ||g||_1^2, Var[v]) per time (Fig. 4b):
    asserts Var[o] <= ||g||_1^2 (1 + slack) at every t — |v| <= 1 bounds
    Var[v] by N_s / (N_s - 1) for the unbiased sample variance, which is the
    default slack."""
    g = np.asarray(g_norm, dtype=np.float64)
    rows = []
    for c, t in enumerate(times):
        var_o = float(stats["var_o"][c, site])
        var_v = float(stats["var_v"][c, site])
        bound = float(g[c] ** 2)
        if slack is None:
            ns = n_samples if n_samples is None or np.ndim(n_samples) == 0 else n_samples[c]
            sl = (1.0 / (ns - 1) if ns and ns > 1 else 0.0) + 1e-12
        else:
            sl = slack
        if var_o > bound * (1.0 + sl):
            raise AssertionError(f"Var[o]={var_o} exceeds ||g||^2={bound} at t={t}")
        rows.append((float(t), var_o, bound, var_v))
    return rows
