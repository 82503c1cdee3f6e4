"""B200-native MLMC level-correction sampler (arXiv 2012.09739 hot path).

The per-level coupled fine/coarse x exact/approximate Euler-Maruyama sampler
and its moment reduction (reference: proj/include/lpmc/{sde,mlmc,stats}.hpp),
as hand-written sm_100a CUDA kernels behind the C-ABI in include/lpmc_b200.h.
This package is the Python mirror of the reference's C++ API; the C++ mirror
lives in include/lpmc/.
"""
from .api import (Allocation, AllocationKind, CostModel, CoupledMoments,  # noqa: F401
                  DomainError, EstimatorResult, InvalidArgument, InvCdfApprox, LevelPlan,
                  LevelStats, MomentAccumulator, PredictedTimes, PrecisionSpec,
                  SamplerRuntimeError, SdeModel, SpeedupResult, allocate_samples, device_count,
                  device_inv_cdf, estimate_level_stats, fold_partials, launch_count,
                  level_partials, level_stats_from_moments, make_gbm, measure_pipe_peaks,
                  per_level_speedup, predicted_times, reset_launch_count, round_to_precision,
                  run_coupled_many, run_coupled_many_partials, run_coupled_paths,
                  run_nested_estimator, run_two_way_paths,
                  simulate_paths, StepErrorStats, step_error_probe, density_histogram)

__all__ = [
    "Allocation", "AllocationKind", "EstimatorResult", "PredictedTimes", "SpeedupResult",
    "allocate_samples", "per_level_speedup", "predicted_times", "run_coupled_many",
    "run_coupled_many_partials",
    "run_nested_estimator", "run_two_way_paths", "StepErrorStats", "step_error_probe", "density_histogram",
    "CostModel", "CoupledMoments", "DomainError", "InvalidArgument", "InvCdfApprox", "LevelPlan",
    "LevelStats", "MomentAccumulator", "PrecisionSpec", "SamplerRuntimeError", "SdeModel",
    "device_count", "device_inv_cdf", "estimate_level_stats", "fold_partials", "launch_count",
    "level_partials", "level_stats_from_moments", "make_gbm", "reset_launch_count",
    "round_to_precision", "run_coupled_paths", "simulate_paths",
]
