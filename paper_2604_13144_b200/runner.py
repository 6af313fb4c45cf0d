"""Cost accounting of an ensemble run (the SPEC's runner cost metrics,
SPEC.md:481-504; PAPER §II.A items 1-3).  The reference package has no runner
module; RunPlan, the worker pool and the CLI stay out
of scope — the ensemble fan-out itself is ``ensemble`` (one GPU) plus
``pipeline_shard`` / ``reduce_pipeline`` (many).

C_circ per sample is measured on the device (``time_samples=True``: the
persistent CTA's globaltimer around the sample) next to the portable proxy
sum_chi_cubed from the per-sample ledger (_kernel.py:150-154)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

COST_COLUMNS = ("sample_id", "nu", "sum_chi_cubed", "wall_ms", "chi_max")


@dataclass
class CostReport:
    """Per-sample circuit costs; TTS = C_tot / N_workers (ideal-parallel model)."""

    sample_ids: np.ndarray
    nu: np.ndarray            # applied unitaries per sample (ledger slot 0)
    sum_chi_cubed: np.ndarray  # proxy cost per sample (ledger slot 1)
    chi_max: np.ndarray
    c_circ: np.ndarray        # measured per-sample cost (ms of device time)
    n_workers: int

    @property
    def c_tot(self) -> float:
        return float(np.sum(self.c_circ))

    @property
    def tts(self) -> float:
        return self.c_tot / self.n_workers

    @property
    def proxy_total(self) -> float:
        return float(np.sum(self.sum_chi_cubed))

    def check(self) -> None:
        """SPEC invariants: TTS * N_workers = C_tot; the deepest sample's
        C_circ <= TTS * N_workers."""
        if abs(self.tts * self.n_workers - self.c_tot) > 1e-9 * max(1.0, self.c_tot):
            raise AssertionError("TTS * N_workers != C_tot")
        if self.c_circ.size and float(np.max(self.c_circ)) > self.tts * self.n_workers * (1 + 1e-12):
            raise AssertionError("deepest C_circ exceeds C_tot")


def cost_report(run, n_workers: int) -> CostReport:
    """CostReport of an ``EnsembleRun`` made with ``time_samples=True``."""
    if n_workers <= 0:
        raise ValueError("n_workers must be positive")
    if run.ledger is None or run.sample_ms is None:
        raise ValueError("per-sample costs not recorded: run the ensemble with time_samples=True")
    ids = run.sample_ids if run.sample_ids is not None else np.arange(run.n_samples)
    rep = CostReport(np.asarray(ids), run.ledger[:, 0].astype(np.int64), run.ledger[:, 1].copy(),
                     run.ledger[:, 2].astype(np.int64), np.asarray(run.sample_ms, dtype=np.float64), int(n_workers))
    rep.check()
    return rep


def tts_tradeoff(report: CostReport, worker_counts, trotter_cost: float | None = None) -> list:
    """Rows (w, TTS(w) = C_tot / w, serial ratio) per requested worker count
    (SPEC.md:497-504): the serial ratio is C_tot / trotter_cost when a
    reference Trotter cost (same units) is supplied, else None."""
    rows = []
    for w in worker_counts:
        if w <= 0:
            raise ValueError("worker count must be positive")
        ratio = report.c_tot / trotter_cost if trotter_cost else None
        rows.append((int(w), report.c_tot / w, ratio))
    return rows


def cost_table(report: CostReport) -> str:
    """Comma-separated cost-report table (SPEC.md:504 columns)."""
    lines = [",".join(COST_COLUMNS)]
    for i in range(report.sample_ids.size):
        lines.append(f"{int(report.sample_ids[i])},{int(report.nu[i])},{float(report.sum_chi_cubed[i])!r},"
                     f"{float(report.c_circ[i])!r},{int(report.chi_max[i])}")
    return "\n".join(lines) + "\n"
