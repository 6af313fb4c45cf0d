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
