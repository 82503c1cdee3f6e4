"""ctypes binding of the C-ABI in include/lpmc_b200.h (liblpmc_b200.so).

The library is the product: every sampling call goes to the sm_100a kernels.
If the library is missing it is built in-tree (nvcc is part of the image); if
that is impossible the import fails loudly.  There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "liblpmc_b200.so")
if os.environ.get("LPMC_LIB"):  # A/B experiments only (build.py --variant=NAME)
    LIB_PATH = os.path.abspath(os.environ["LPMC_LIB"])

_u64 = C.c_uint64
_i32 = C.c_int32
_dp = C.POINTER(C.c_double)

LPMC_OK = 0
LPMC_INVALID_ARGUMENT = 1
LPMC_DOMAIN_ERROR = 2
LPMC_RUNTIME_ERROR = 3
LPMC_CUDA_ERROR = 4
LPMC_NO_DEVICE = 5

LEGS_HAT, LEGS_BAR, LEGS_ALL, LEGS_FINE = 1, 2, 3, 4
ALLOCATION_STANDARD, ALLOCATION_NESTED = 0, 1
PAYOFF_TERMINAL, PAYOFF_CALL = 0, 1
REDUCE_TREE, REDUCE_SEQUENTIAL = 0, 1
EXACT_Z_FAST, EXACT_Z_GLIBC = 0, 1
SCHEDULE_AUTO, SCHEDULE_FUSED, SCHEDULE_WARP_PER_PATH = 0, 1, 2
APPROX_LINEAR, APPROX_CUBIC, APPROX_CONSTANT = 0, 1, 2
BATCH_PATHS = 256
CHUNK_BATCHES = 1024
CHUNK_PATHS = BATCH_PATHS * CHUNK_BATCHES


class LpmcError(Exception):
    """Base of the errors the C-ABI reports."""


class InvalidArgument(LpmcError, ValueError):
    """std::invalid_argument in the reference."""


class DomainError(LpmcError, ValueError):
    """std::domain_error in the reference."""


class SamplerRuntimeError(LpmcError, RuntimeError):
    """std::runtime_error in the reference."""


class CudaError(LpmcError, RuntimeError):
    """Device or driver failure (no reference counterpart; never masked)."""


class NoDevice(CudaError):
    """No sm_100 device visible."""


_ERRORS = {LPMC_INVALID_ARGUMENT: InvalidArgument, LPMC_DOMAIN_ERROR: DomainError,
           LPMC_RUNTIME_ERROR: SamplerRuntimeError, LPMC_CUDA_ERROR: CudaError,
           LPMC_NO_DEVICE: NoDevice}


class Error(C.Structure):
    _fields_ = [("status", _i32), ("kind", _i32), ("path_index", _u64), ("step", _u64),
                ("message", C.c_char * 192)]


class Gbm(C.Structure):
    _fields_ = [("mu", C.c_double), ("sigma", C.c_double), ("x0", C.c_double),
                ("horizon", C.c_double)]


class InvCdfTable(C.Structure):
    _fields_ = [("kind", _i32), ("interval_count", _i32), ("w_max", C.c_double),
                ("step_w", C.c_double), ("tail_value", C.c_double), ("breakpoints", _dp),
                ("coeff", _dp)]


class Precision(C.Structure):
    _fields_ = [("mantissa_bits", _i32), ("ieee_half", _i32)]


class Options(C.Structure):
    _fields_ = [("legs", C.c_uint32), ("payoff", _i32), ("strike", C.c_double),
                ("reduce", _i32), ("device", _i32), ("stream", C.c_void_p),
                ("exact_z", _i32), ("devices", C.POINTER(_i32)), ("n_devices", _i32),
                ("schedule", _i32), ("counter", _u64)]


class Moments(C.Structure):
    _fields_ = [("n", _u64), ("mean", C.c_double), ("m2", C.c_double), ("m3", C.c_double),
                ("m4", C.c_double)]

    def as_tuple(self):
        return (int(self.n), self.mean, self.m2, self.m3, self.m4)


class CostModelC(C.Structure):
    _fields_ = [("cycles_exact_rng", C.c_double), ("cycles_approx_rng_single", C.c_double),
                ("cycles_approx_rng_half", C.c_double), ("kahan_overhead_factor", C.c_double),
                ("per_step_arithmetic", C.c_double)]


class LevelStatsC(C.Structure):
    _fields_ = [("level", _i32), ("mean_hat", C.c_double), ("v_hat", C.c_double),
                ("v_hat_stderr", C.c_double), ("mean_bar", C.c_double), ("v_bar", C.c_double),
                ("v_bar_stderr", C.c_double), ("mean_four", C.c_double), ("V_bar", C.c_double),
                ("V_bar_stderr", C.c_double), ("c_hat", C.c_double), ("c_bar", C.c_double),
                ("C_bar", C.c_double), ("m_hat", _u64), ("m_bar", _u64), ("M_bar", _u64)]


class RunDesc(C.Structure):
    _fields_ = [("level", _i32), ("prec", Precision), ("kahan", _i32), ("n_paths", _u64),
                ("path_base", _u64)]


class EstimatorResultC(C.Structure):
    _fields_ = [("value", C.c_double), ("eps", C.c_double), ("t_hat", C.c_double),
                ("t_bar", C.c_double), ("degenerate", _i32), ("level_contributions", _dp),
                ("pilot_stats", C.POINTER(LevelStatsC)), ("primary", C.POINTER(_u64)),
                ("secondary", C.POINTER(_u64))]


class StepErrorStatsC(C.Structure):
    _fields_ = [("mean_eta", C.c_double), ("mean_abs_eta", C.c_double),
                ("mean_eta_prime", C.c_double), ("mean_abs_eta_prime", C.c_double),
                ("samples", _u64)]


# exported symbol -> (restype, argtypes); the CPU test suite checks every
# symbol include/lpmc_b200.h declares is exported and bound here.
_P = C.POINTER
SIGNATURES = {
    "lpmc_abi_version": (_i32, []),
    "lpmc_device_count": (_i32, []),
    "lpmc_launch_count": (_u64, []),
    "lpmc_reset_launch_count": (None, []),
    "lpmc_default_options": (None, [_P(Options)]),
    "lpmc_default_cost_model": (None, [_P(CostModelC)]),
    "lpmc_round_to_precision": (_i32, [C.c_double, _i32, _dp, _P(Error)]),
    "lpmc_invcdf_build": (_i32, [_i32, _i32, _dp, _dp, _dp, _dp, _dp, _P(Error)]),
    "lpmc_invcdf_eval": (_i32, [_P(InvCdfTable), C.c_double, _dp, _P(Error)]),
    "lpmc_moments_add": (None, [_P(Moments), C.c_double]),
    "lpmc_moments_merge": (None, [_P(Moments), _P(Moments)]),
    "lpmc_fold_partials": (None, [_P(Moments), _u64, _P(Moments)]),
    "lpmc_level_stats_from_moments": (None, [_P(Moments), _i32, _P(Precision), _i32,
                                             _P(CostModelC), _u64, _P(LevelStatsC)]),
    "lpmc_run_coupled_paths": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32, _u64,
                                      _u64, _u64, _P(Options), _P(Moments), _P(Error)]),
    "lpmc_estimate_level_stats": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32,
                                         _u64, _u64, _P(CostModelC), _u64, _P(Options),
                                         _P(LevelStatsC), _P(Error)]),
    "lpmc_level_partials": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32, _u64,
                                   _u64, _u64, _u64, _u64, _P(Options), _P(Moments),
                                   _P(Error)]),
    "lpmc_simulate_paths": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32, _u64,
                                   _u64, _u64, _P(Options), _dp, _dp, _P(Error)]),
    "lpmc_device_inv_cdf": (_i32, [_dp, _u64, _P(InvCdfTable), _dp, _P(Options), _P(Error)]),
    "lpmc_measure_pipe_peaks": (_i32, [_i32, _dp, _P(Error)]),
    "lpmc_device_math": (_i32, [_i32, _dp, _u64, _P(InvCdfTable), _dp, _P(Options), _P(Error)]),
    "lpmc_bar_arithmetic": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32,
                                   _P(Options), _P(_i32), _P(Error)]),
    "lpmc_erfc_core": (C.c_double, [C.c_double]),
    "lpmc_phi_inv_direct_core": (C.c_double, [C.c_double, _P(_i32)]),
    "lpmc_glibc_math": (C.c_double, [_i32, C.c_double, _P(_i32)]),
    "lpmc_run_coupled_many": (_i32, [_P(Gbm), _P(InvCdfTable), _u64, _P(RunDesc), _u64,
                                     _P(Options), _P(Moments), _P(Error)]),
    "lpmc_run_coupled_many_partials": (_i32, [_P(Gbm), _P(InvCdfTable), _u64, _P(RunDesc), _u64,
                                              _P(_u64), _P(_u64), _P(Options), _P(Moments),
                                              _P(Error)]),
    "lpmc_stream_word": (_u64, [_u64, _u64, _u64]),
    "lpmc_stream_uniform": (C.c_double, [_u64, _u64, _u64]),
    "lpmc_normal_cdf": (C.c_double, [C.c_double]),
    "lpmc_normal_pdf": (C.c_double, [C.c_double]),
    "lpmc_exact_inv_cdf": (_i32, [C.c_double, _dp, _P(Error)]),
    "lpmc_inv_cdf_lower": (C.c_double, [C.c_double]),
    "lpmc_gauss_legendre": (_i32, [_i32, _dp, _dp, _P(Error)]),
    "lpmc_ulp_spacing": (_i32, [C.c_double, _i32, _dp, _P(Error)]),
    "lpmc_moment_diagnostics": (_i32, [_P(InvCdfTable), _i32, _dp, _P(Error)]),
    "lpmc_run_two_way_paths": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32, _u64,
                                      _u64, _u64, _P(Options), _P(Moments), _P(Error)]),
    "lpmc_allocate_samples": (_i32, [_P(LevelStatsC), _u64, C.c_double, _i32, _P(_u64),
                                     _P(_u64), _P(_i32), _P(Error)]),
    "lpmc_predicted_times": (_i32, [_P(LevelStatsC), _u64, C.c_double, _dp, _dp, _P(Error)]),
    "lpmc_per_level_speedup": (_i32, [_P(LevelStatsC), _dp, _P(_i32), _P(Error)]),
    "lpmc_run_nested_estimator": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32,
                                         C.c_double, _u64, _P(CostModelC), _u64, _P(Options),
                                         _P(EstimatorResultC), _P(Error)]),
    "lpmc_density_histogram": (_i32, [_P(InvCdfTable), _u64, _u64, C.c_double, C.c_double, _i32,
                                      _P(_u64), _P(Options), _P(Error)]),
    "lpmc_step_error_probe": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _u64, _u64,
                                     _P(Options), _P(StepErrorStatsC), _P(Error)]),
    "lpmc_plan_create": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32, _u64, _u64,
                                _u64, _P(Options), _P(C.c_void_p), _P(Error)]),
    "lpmc_plan_create_range": (_i32, [_P(Gbm), _i32, _P(Precision), _P(InvCdfTable), _i32, _u64,
                                      _u64, _u64, _u64, _u64, _P(Options), _P(C.c_void_p),
                                      _P(Error)]),
    "lpmc_plan_launch": (_i32, [C.c_void_p, C.c_void_p, _P(Error)]),
    "lpmc_plan_collect_partials": (_i32, [C.c_void_p, _P(Moments), _P(Error)]),
    "lpmc_plan_chunk_count": (_u64, [C.c_void_p]),
    "lpmc_plan_collect": (_i32, [C.c_void_p, _P(Moments), _P(Error)]),
    "lpmc_plan_kernels_per_launch": (_i32, [C.c_void_p]),
    "lpmc_plan_destroy": (None, [C.c_void_p]),
}

_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load liblpmc_b200.so (building it in-tree first if it is missing)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if not build_if_missing:
                raise ImportError(f"{LIB_PATH} is missing; run python -m paper_2012_09739_b200.build")
            from . import build as _build
            _build.build()
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.lpmc_abi_version() != 3:
            raise ImportError("liblpmc_b200.so ABI version mismatch")
        _lib = lib
        return lib


def check(status: int, err: Error) -> None:
    if status == LPMC_OK:
        return
    cls = _ERRORS.get(status, LpmcError)
    exc = cls(err.message.decode(errors="replace"))
    exc.kind = int(err.kind)
    exc.path_index = int(err.path_index)
    exc.step = int(err.step)
    raise exc


def default_options(**kw) -> Options:
    o = Options()
    load().lpmc_default_options(C.byref(o))
    for k, v in kw.items():
        if v is not None:
            setattr(o, k, v)
    return o
