"""B200-native MPS sampling sweep (FastMPS, arxiv 2512.20064).

The hot path — contract L[N, chi] x Gamma_i, Born weights, keyed draw, gather + renormalise — runs
in hand-written sm_100a kernels (libmpsg.so, tcgen05/TMEM/TMA) behind the C ABI in
include/mpsg.h.  This package is the host-side mirror of the reference's ``mpsamp`` interface.
"""
from .sampler import (  # noqa: F401
    DEAD_OUTCOME,
    BatchPlan,
    BondSchedule,
    ParallelResult,
    apply_schedule,
    dynamic_bond_schedule,
    entanglement_entropy,
    TruncationFilter,
    run_data_parallel,
    run_serial,
    ConfigError,
    DeviceError,
    DimensionError,
    Displacement,
    Error,
    GpuSampler,
    IoError,
    Mode,
    MpsState,
    NumericError,
    Precision,
    PrecisionPolicy,
    RunStats,
    SampleBatch,
    SamplerOptions,
    ScalingMode,
    Scheme,
    Slice,
    capped_bond_dims,
    decay_probe,
    device_draws,
    displacement_matrix,
    sample_batch,
    sample_micro_serial,
)
