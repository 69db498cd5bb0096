"""B200-native batched Kaczmarz RZF precoding (arXiv 2501.10689 hot path).

Drop-in for the solver path of the reference package `kaczprec`
(pkg/src/kaczprec/__init__.py:69-131): the same public names for the solver,
RZF, assembly and metric entry points, backed by libkaczmarz_b200.so
(hand-written sm_100a CUDA behind the C ABI in include/kaczmarz_b200.h).
Batched entry points (`solve_batch`, `run_precoding_batched`, `rzf_batched`,
`epilogue`) run thousands of systems per launch.  There is no CPU fallback.
"""

from .assembly import SubarrayChannel, assemble_dense, assemble_vr, epilogue
from .batch import DeviceBatch, HostBatch, pin_host
from .channel import CONFIGS, ContiguousChannels, Drops, NearFieldConfig, generate, generate_drops, solver_seed_sequence
from .metrics import CADD, CMUL, nmse, spectral_efficiency
from .rzf import Precoder, apply_auxiliary, auxiliary_matrix, mrc_precoder, rzf_batched, rzf_precoder
from .solvers import (
    SCHEMES,
    EXTENDED_SCHEMES,
    AggregationWeights,
    InstanceRun,
    SelectionStrategy,
    ahk_step,
    aggregation_weights,
    orthogonal_block_step,
    residual_refresh,
    rk_step,
    select_row,
    STOCHASTIC_SCHEMES,
    VR_SCHEMES,
    AugmentedSystem,
    BatchResult,
    FlopCounter,
    HostStreams,
    PrecodingRun,
    RunTrace,
    SolverState,
    StoppingRule,
    canonical_scheme,
    display_scheme,
    run_precoding,
    run_precoding_batched,
    solve,
    solve_all,
    solve_batch,
)
from .shard import gather_stats, shard_range
from .vrgraph import UserPartition, build_partition

__version__ = "0.1.0"

__all__ = [
    "AugmentedSystem", "BatchResult", "CADD", "CMUL", "CONFIGS", "ContiguousChannels", "DeviceBatch", "Drops",
    "FlopCounter", "HostBatch", "HostStreams", "NearFieldConfig", "Precoder", "PrecodingRun", "RunTrace",
    "SCHEMES", "EXTENDED_SCHEMES", "STOCHASTIC_SCHEMES", "SolverState", "StoppingRule", "UserPartition", "VR_SCHEMES",
    "apply_auxiliary", "assemble_dense", "assemble_vr", "auxiliary_matrix", "build_partition",
    "canonical_scheme", "display_scheme", "epilogue", "generate", "generate_drops", "mrc_precoder", "nmse", "pin_host", "rzf_batched",
    "rzf_precoder", "run_precoding", "run_precoding_batched", "solve", "solve_all", "solve_batch",
    "solver_seed_sequence", "spectral_efficiency", "gather_stats", "shard_range",
    "AggregationWeights", "InstanceRun", "SubarrayChannel", "SelectionStrategy", "ahk_step", "aggregation_weights",
    "orthogonal_block_step", "residual_refresh", "rk_step", "select_row",
]
