"""B200-native MPS TE-PAI ensemble engine (drop-in for the reference ``tepai``
package's hot path: sampler -> MPS simulation -> signed weighted estimator).

Public names mirror ``pkg/src/tepai/__init__.py:11-52`` for the path in scope
plus the batched ``run_ensemble`` / ``aggregate`` of SPEC.md.
"""

from .estimator import (
    EnsembleResult,
    SampleRecord,
    SignedMixture,
    aggregate,
    aggregate_fixed,
    evaluate_observables,
    mixture_from_run,
    per_sample_expectations,
    results_table,
    variance_vs_bound_trace,
)
from .runner import CostReport, cost_report, cost_table, tts_tradeoff
from .ensemble import (
    SlotPipeline,
    EnsembleRun,
    PackedEnsemble,
    allreduce_sums,
    broadcast_state,
    run_hybrid,
    checkpoint_weights,
    pack_ensemble,
    run_ensemble,
    run_packed,
    shard_range,
    pipeline_shard,
    reduce_pipeline,
)
from .mps import (
    EXACT,
    CostLedger,
    MPSState,
    TruncationPolicy,
    apply_pauli_rotation,
    discarded_weight,
    expectation,
    init_product_state,
    load_snapshot,
    max_bond,
    run_circuit,
    save_snapshot,
    snapshot_from_bytes,
    snapshot_to_bytes,
)
from .pauli import Hamiltonian, HamTerm, PauliString, build_spin_ring, build_tfim_ring, coeff_l1_norm, min_trotter_steps
from .rng import circuit_stream, disorder_stream, philox_stream
from .sampling import (
    PaiConfig,
    SampledCircuit,
    circuit_weight_norm,
    expected_gate_count_inf,
    gamma_coeffs,
    gamma_l1_norm,
    overhead_norm_inf,
    sample_circuit,
    variant_probabilities,
)
from .trotter import TrotterCircuit, build_trotter_circuit

__version__ = "0.1.0"
