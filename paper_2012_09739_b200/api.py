"""Python mirror of the reference's level-sampling API (proj/include/lpmc).

Same names, argument meaning and error behaviour as the C++ reference, so the
parity tests read like the reference's own tests:

==========================  ================================================
this module                 reference (/root/reference/proj/include/lpmc)
==========================  ================================================
PrecisionSpec               softfloat.hpp:18-64
round_to_precision          softfloat.hpp:69-80
InvCdfApprox                invcdf_approx.hpp:28-145 (+ ``constant:K``)
SdeModel / make_gbm         sde.hpp:24-44
MomentAccumulator           stats.hpp:13-90
CoupledMoments              mlmc.hpp:53-63
CostModel / LevelStats      mlmc.hpp:20-51
run_coupled_paths           mlmc.hpp:67-111   (device: lpmc_run_coupled_paths)
estimate_level_stats        mlmc.hpp:113-149  (device: lpmc_estimate_level_stats)
run_two_way_paths           experiments.hpp:136-141 over sde.hpp:162-196
                            (device: lpmc_run_two_way_paths)
AllocationKind/Allocation,  mlmc.hpp:151-195
allocate_samples
PredictedTimes,             mlmc.hpp:197-213
predicted_times
SpeedupResult,              mlmc.hpp:215-230
per_level_speedup
EstimatorResult,            mlmc.hpp:232-283  (device: lpmc_run_nested_estimator)
run_nested_estimator
StepErrorStats,             sde.hpp:289-344   (device: lpmc_step_error_probe)
step_error_probe
==========================  ================================================

Every sampling call runs on the sm_100a kernels through the C-ABI; there is
no CPU path.  Exceptions: InvalidArgument (std::invalid_argument),
DomainError (std::domain_error), SamplerRuntimeError (std::runtime_error).

Extensions beyond the reference (keyword-only, defaults reproduce the
reference): ``legs`` (hat/bar/all), ``payoff`` ("terminal" | "call") with
``strike``, ``reduce`` ("tree" | "sequential"), ``device``, ``stream``, and
``PrecisionSpec.fp16_ieee()`` for native IEEE-binary16 legs.  ``legs="fine"``
runs the two-way sampler (fine legs only); ``run_coupled_many`` runs a list of
levels concurrently on one device.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N
from ._native import DomainError, InvalidArgument, SamplerRuntimeError  # noqa: F401

_LEGS = {"hat": N.LEGS_HAT, "bar": N.LEGS_BAR, "all": N.LEGS_ALL, "fine": N.LEGS_FINE}
_PAYOFF = {"terminal": N.PAYOFF_TERMINAL, "call": N.PAYOFF_CALL}
_REDUCE = {"tree": N.REDUCE_TREE, "sequential": N.REDUCE_SEQUENTIAL}
# exact Gaussians: "fast" (B200 restatement, ulp-level) or "glibc" (the
# reference's Z bit for bit, lpmc_glibc.cuh)
_EXACT_Z = {"fast": N.EXACT_Z_FAST, "glibc": N.EXACT_Z_GLIBC}
_SCHEDULE = {"auto": N.SCHEDULE_AUTO, "fused": N.SCHEDULE_FUSED,
             "warp_per_path": N.SCHEDULE_WARP_PER_PATH}


# ----------------------------------------------------------- precision -----
@dataclass(frozen=True)
class PrecisionSpec:
    """Stored fraction bits (softfloat.hpp:18-64); ieee_half selects native
    IEEE binary16 legs (extension, BASELINE config 3)."""

    mantissa_bits: int
    ieee_half: bool = False

    kMaxMantissaBits = 26
    kCarrierMantissaBits = 52

    def unit_roundoff(self) -> float:
        return math.ldexp(1.0, -(self.mantissa_bits + 1))

    def is_carrier(self) -> bool:
        return self.mantissa_bits >= self.kCarrierMantissaBits

    @staticmethod
    def bf16():
        return PrecisionSpec(7)

    @staticmethod
    def fp16():
        return PrecisionSpec(10)

    @staticmethod
    def fp16_ieee():
        return PrecisionSpec(10, True)

    @staticmethod
    def fp22():
        return PrecisionSpec(16)

    @staticmethod
    def fp32():
        return PrecisionSpec(23)

    @staticmethod
    def carrier():
        return PrecisionSpec(52)

    @staticmethod
    def custom(m: int):
        if m < 1 or m > PrecisionSpec.kMaxMantissaBits:
            raise InvalidArgument(f"mantissa_bits must be in [1, 26], got {m}")
        return PrecisionSpec(m)

    @staticmethod
    def parse(name: str) -> "PrecisionSpec":
        table = {"bf16": 7, "fp16": 10, "fp22": 16, "fp32": 23, "carrier": 52, "fp64": 52,
                 "double": 52}
        if name in table:
            return PrecisionSpec(table[name])
        if name == "fp16-ieee":
            return PrecisionSpec.fp16_ieee()
        if name.startswith("custom:"):
            try:
                m = int(name[7:])
            except ValueError:
                raise InvalidArgument(f"bad precision name: {name}") from None
            return PrecisionSpec.custom(m)
        raise InvalidArgument(f"bad precision name: {name}")

    def _c(self) -> N.Precision:
        return N.Precision(self.mantissa_bits, int(self.ieee_half))


def round_to_precision(x: float, spec: PrecisionSpec) -> float:
    out = C.c_double()
    err = N.Error()
    N.check(N.load().lpmc_round_to_precision(float(x), spec.mantissa_bits, C.byref(out),
                                             C.byref(err)), err)
    return out.value


# ------------------------------------------------------ approximations -----
class InvCdfApprox:
    """Piecewise-polynomial inverse normal CDF (invcdf_approx.hpp:28-145).

    Built on the host by the library (bitwise the reference's table); the
    device receives it per call.  ``constant:K`` is the degree-0 extension.
    """

    KINDS = {"linear": N.APPROX_LINEAR, "cubic": N.APPROX_CUBIC, "constant": N.APPROX_CONSTANT}

    def __init__(self, kind: str, K: int, w_max: float, step_w: float, tail: float,
                 breakpoints: np.ndarray, coeff: np.ndarray):
        self.kind = kind
        self._K = K
        self.w_max = w_max
        self.step_w = step_w
        self.tail_value = tail
        self._bp = np.ascontiguousarray(breakpoints, dtype=np.float64)
        self._coeff = np.ascontiguousarray(coeff, dtype=np.float64).reshape(K, 4)
        self._c = N.InvCdfTable(self.KINDS[kind], K, w_max, step_w, tail,
                                self._bp.ctypes.data_as(N._dp),
                                self._coeff.ctypes.data_as(N._dp))

    _built: dict = {}  # (kind, K) -> table: builds are deterministic, tables immutable

    @classmethod
    def build(cls, kind: str, interval_count: int) -> "InvCdfApprox":
        if kind not in cls.KINDS:
            raise InvalidArgument(f"bad approximation kind: {kind}")
        K = int(interval_count)
        if K < 2 or (K & (K - 1)) != 0:
            raise InvalidArgument("interval count must be a power of two >= 2")
        hit = cls._built.get((kind, K))
        if hit is not None:
            return hit
        bp = np.zeros(K)
        co = np.zeros(4 * K)
        wm, sw, tl = C.c_double(), C.c_double(), C.c_double()
        err = N.Error()
        N.check(N.load().lpmc_invcdf_build(cls.KINDS[kind], K, bp.ctypes.data_as(N._dp),
                                           co.ctypes.data_as(N._dp), C.byref(wm), C.byref(sw),
                                           C.byref(tl), C.byref(err)), err)
        table = cls(kind, K, wm.value, sw.value, tl.value, bp, co)
        bp.flags.writeable = False
        co.flags.writeable = False
        table._bp.flags.writeable = False
        table._coeff.flags.writeable = False
        cls._built[(kind, K)] = table
        return table

    @classmethod
    def parse(cls, name: str) -> "InvCdfApprox":
        kind, sep, k = name.partition(":")
        if not sep:
            raise InvalidArgument(f"bad approximation name: {name}")
        try:
            K = int(k)
        except ValueError:
            raise InvalidArgument(f"bad approximation name: {name}") from None
        if kind not in cls.KINDS:
            raise InvalidArgument(f"bad approximation name: {name}")
        return cls.build(kind, K)

    def interval_count(self) -> int:
        return self._K

    def degree(self) -> int:
        return {"linear": 1, "cubic": 3, "constant": 0}[self.kind]

    def breakpoints(self) -> np.ndarray:
        return self._bp

    def coefficients(self) -> np.ndarray:
        return self._coeff

    def truncation_point(self) -> float:
        return float(self._bp[-1])

    def max_value(self) -> float:
        return self.tail_value

    def __call__(self, u: float) -> float:
        out = C.c_double()
        err = N.Error()
        N.check(N.load().lpmc_invcdf_eval(C.byref(self._c), float(u), C.byref(out),
                                          C.byref(err)), err)
        return out.value

    @property
    def c_table(self) -> N.InvCdfTable:
        return self._c


# ------------------------------------------------------------ models -------
@dataclass
class SdeModel:
    """sde.hpp:24-30.  The device sampler needs the GBM parameters, so
    make_gbm tags the model; any other model is rejected (no CPU fallback)."""

    drift: Optional[Callable] = None
    diffusion: Optional[Callable] = None
    x0: float = 1.0
    horizon: float = 1.0
    gbm: Optional[tuple] = None  # (mu, sigma) when built by make_gbm


def make_gbm(mu: float = 0.05, sigma: float = 0.2, x0: float = 1.0,
             horizon: float = 1.0) -> SdeModel:
    def drift(t, x, spec):
        return round_to_precision(round_to_precision(mu, spec) * x, spec)

    def diffusion(t, x, spec):
        return round_to_precision(round_to_precision(sigma, spec) * x, spec)

    return SdeModel(drift, diffusion, x0, horizon, (mu, sigma))


def _gbm_c(model: SdeModel) -> N.Gbm:
    if model.gbm is None:
        raise InvalidArgument("the device sampler supports GBM models built by make_gbm")
    mu, sigma = model.gbm
    return N.Gbm(mu, sigma, model.x0, model.horizon)


# ------------------------------------------------------------ moments ------
@dataclass
class MomentAccumulator:
    """Raw central-moment state (stats.hpp:13-90); add/merge are the
    library's bitwise restatements."""

    n: int = 0
    mean_: float = 0.0
    m2: float = 0.0
    m3: float = 0.0
    m4: float = 0.0

    @classmethod
    def from_c(cls, m: N.Moments) -> "MomentAccumulator":
        return cls(int(m.n), m.mean, m.m2, m.m3, m.m4)

    def to_c(self) -> N.Moments:
        return N.Moments(self.n, self.mean_, self.m2, self.m3, self.m4)

    def add(self, x: float) -> None:
        c = self.to_c()
        N.load().lpmc_moments_add(C.byref(c), float(x))
        self.n, self.mean_, self.m2, self.m3, self.m4 = c.as_tuple()

    def merge(self, other: "MomentAccumulator") -> None:
        a, b = self.to_c(), other.to_c()
        N.load().lpmc_moments_merge(C.byref(a), C.byref(b))
        self.n, self.mean_, self.m2, self.m3, self.m4 = a.as_tuple()

    def count(self) -> int:
        return self.n

    def mean(self) -> float:
        return self.mean_ if self.n else 0.0

    def variance(self) -> float:
        return self.m2 / (self.n - 1) if self.n >= 2 else 0.0

    def fourth_central_moment(self) -> float:
        return self.m4 / self.n if self.n else 0.0

    def variance_stderr(self) -> float:
        if self.n < 2:
            return 0.0
        v = self.variance()
        spread = max(self.fourth_central_moment() - v * v, 0.0)
        return math.sqrt(spread / self.n)

    def mean_stderr(self) -> float:
        return math.sqrt(self.variance() / self.n) if self.n >= 2 else 0.0

    def state(self) -> tuple:
        return (self.n, self.mean_, self.m2, self.m3, self.m4)


@dataclass
class CoupledMoments:
    d_hat: MomentAccumulator = field(default_factory=MomentAccumulator)
    d_bar: MomentAccumulator = field(default_factory=MomentAccumulator)
    d_four: MomentAccumulator = field(default_factory=MomentAccumulator)

    def merge(self, other: "CoupledMoments") -> None:
        self.d_hat.merge(other.d_hat)
        self.d_bar.merge(other.d_bar)
        self.d_four.merge(other.d_four)

    @classmethod
    def from_c3(cls, acc) -> "CoupledMoments":
        return cls(*(MomentAccumulator.from_c(acc[i]) for i in range(3)))


@dataclass
class CostModel:
    cycles_exact_rng: float = 3.5
    cycles_approx_rng_single: float = 0.5
    cycles_approx_rng_half: float = 0.25
    kahan_overhead_factor: float = 1.4
    per_step_arithmetic: float = 0.0

    def approx_rng_cycles(self, spec: PrecisionSpec) -> float:
        return self.cycles_approx_rng_half if spec.mantissa_bits <= 10 else \
            self.cycles_approx_rng_single

    def _c(self) -> N.CostModelC:
        return N.CostModelC(self.cycles_exact_rng, self.cycles_approx_rng_single,
                            self.cycles_approx_rng_half, self.kahan_overhead_factor,
                            self.per_step_arithmetic)


@dataclass
class LevelStats:
    level: int = 0
    mean_hat: float = 0.0
    v_hat: float = 0.0
    v_hat_stderr: float = 0.0
    mean_bar: float = 0.0
    v_bar: float = 0.0
    v_bar_stderr: float = 0.0
    mean_four: float = 0.0
    V_bar: float = 0.0
    V_bar_stderr: float = 0.0
    c_hat: float = 0.0
    c_bar: float = 0.0
    C_bar: float = 0.0
    m_hat: int = 0
    m_bar: int = 0
    M_bar: int = 0

    @classmethod
    def from_c(cls, s: N.LevelStatsC) -> "LevelStats":
        return cls(**{name: getattr(s, name) for name, _ in N.LevelStatsC._fields_})

    def _c(self) -> N.LevelStatsC:
        return N.LevelStatsC(**{name: getattr(self, name) for name, _ in N.LevelStatsC._fields_})


# ------------------------------------------------------------ sampling -----
def _options(legs="all", payoff="terminal", strike=1.0, reduce="tree", device=None,
             stream=None, exact_z="fast", devices=None, schedule="auto") -> N.Options:
    """Per-call options.  ``devices``: several CUDA ordinals of this process
    to shard each run over (chunk ranges, folded in chunk order: bitwise the
    single-device result); the call is then synchronous.  ``schedule``:
    "auto", "fused" or "warp_per_path" (results identical)."""
    try:
        o = N.default_options(legs=_LEGS[legs], payoff=_PAYOFF[payoff], strike=float(strike),
                              reduce=_REDUCE[reduce],
                              device=-1 if device is None else int(device),
                              stream=None if stream is None else int(stream),
                              exact_z=_EXACT_Z[exact_z], schedule=_SCHEDULE[schedule])
    except KeyError as e:
        raise InvalidArgument(f"bad option value {e}") from None
    if devices is not None and len(devices) > 0:
        o._devices = (C.c_int32 * len(devices))(*[int(d) for d in devices])  # kept alive
        o.devices = C.cast(o._devices, C.POINTER(C.c_int32))
        o.n_devices = len(devices)
    return o


def _table_ptr(approx: Optional[InvCdfApprox]):
    return None if approx is None else C.byref(approx.c_table)


def run_coupled_paths(model: SdeModel, level: int, spec_low: PrecisionSpec,
                      approx: Optional[InvCdfApprox], kahan: bool, n_paths: int, seed: int,
                      path_base: int, threads: int = 1, **ext) -> CoupledMoments:
    """mlmc.hpp:67-111 on the device.  ``threads`` only scheduled the CPU
    reference and never changed its result; it is accepted and ignored."""
    acc = (N.Moments * 3)()
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_run_coupled_paths(C.byref(_gbm_c(model)), int(level),
                                            C.byref(spec_low._c()), _table_ptr(approx),
                                            int(bool(kahan)), int(n_paths), int(seed),
                                            int(path_base), C.byref(opts), acc, C.byref(err)),
            err)
    return CoupledMoments.from_c3(acc)


def estimate_level_stats(model: SdeModel, level: int, spec_low: PrecisionSpec,
                         approx: Optional[InvCdfApprox], kahan: bool, n_paths: int, seed: int,
                         cost: Optional[CostModel] = None, threads: int = 1, path_base: int = 0,
                         **ext) -> LevelStats:
    """mlmc.hpp:113-149 on the device."""
    out = N.LevelStatsC()
    err = N.Error()
    opts = _options(**ext)
    cm = (cost or CostModel())._c()
    N.check(N.load().lpmc_estimate_level_stats(C.byref(_gbm_c(model)), int(level),
                                               C.byref(spec_low._c()), _table_ptr(approx),
                                               int(bool(kahan)), int(n_paths), int(seed),
                                               C.byref(cm), int(path_base), C.byref(opts),
                                               C.byref(out), C.byref(err)), err)
    return LevelStats.from_c(out)


def run_coupled_many(model: SdeModel, approx: Optional[InvCdfApprox], seed: int, runs,
                     **ext) -> list:
    """Several run_coupled_paths calls (same model, table, seed and options)
    executed concurrently on one device; ``runs`` holds (level, spec_low,
    kahan, n_paths, path_base) tuples.  Returns one CoupledMoments per run,
    bitwise those of the separate calls; the first failing run in list order
    raises, as a serial loop would."""
    runs = list(runs)
    descs = (N.RunDesc * max(1, len(runs)))()
    for i, (level, spec, kahan, n, base) in enumerate(runs):
        descs[i] = N.RunDesc(int(level), spec._c(), int(bool(kahan)), int(n), int(base))
    acc = (N.Moments * max(1, 3 * len(runs)))()
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_run_coupled_many(C.byref(_gbm_c(model)), _table_ptr(approx), int(seed),
                                           descs, len(runs), C.byref(opts), acc, C.byref(err)),
            err)
    return [CoupledMoments.from_c3(acc[3 * i:3 * i + 3]) for i in range(len(runs))]


def run_coupled_many_partials(model: SdeModel, approx: Optional[InvCdfApprox], seed: int, runs,
                              chunk_ranges, **ext) -> list:
    """run_coupled_many over one chunk range per run (this rank's shard):
    ``chunk_ranges`` holds (chunk_begin, chunk_end) per run.  Returns one
    (k_i, 3, 5) array of raw chunk accumulators per run (fold the gathered
    shards of all ranks with fold_partials)."""
    runs = list(runs)
    ranges = [(int(a), int(b)) for a, b in chunk_ranges]
    if len(ranges) != len(runs):
        raise InvalidArgument("one chunk range per run")
    n = max(1, len(runs))
    descs = (N.RunDesc * n)()
    cb = (C.c_uint64 * n)()
    ce = (C.c_uint64 * n)()
    for i, (level, spec, kahan, npaths, base) in enumerate(runs):
        descs[i] = N.RunDesc(int(level), spec._c(), int(bool(kahan)), int(npaths), int(base))
        cb[i], ce[i] = ranges[i]
    total = sum(max(b - a, 0) for a, b in ranges)
    acc = (N.Moments * max(1, 3 * total))()
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_run_coupled_many_partials(C.byref(_gbm_c(model)), _table_ptr(approx),
                                                    int(seed), descs, len(runs), cb, ce,
                                                    C.byref(opts), acc, C.byref(err)), err)
    flat = np.array([acc[i].as_tuple() for i in range(3 * total)],
                    dtype=np.float64).reshape(-1, 3, 5)
    out, o = [], 0
    for a, b in ranges:
        k = max(b - a, 0)
        out.append(flat[o:o + k])
        o += k
    return out


def run_two_way_paths(model: SdeModel, level: int, spec_low: PrecisionSpec,
                      approx: Optional[InvCdfApprox], kahan: bool, n_paths: int, seed: int,
                      path_base: int, threads: int = 1, **ext) -> MomentAccumulator:
    """MomentAccumulator of x_hat - x_bar over simulate_two_way paths
    (sde.hpp:162-196), merged like run_batched (experiments.hpp:89-112)."""
    out = N.Moments()
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_run_two_way_paths(C.byref(_gbm_c(model)), int(level),
                                            C.byref(spec_low._c()), _table_ptr(approx),
                                            int(bool(kahan)), int(n_paths), int(seed),
                                            int(path_base), C.byref(opts), C.byref(out),
                                            C.byref(err)), err)
    return MomentAccumulator.from_c(out)


def level_stats_from_moments(m: CoupledMoments, level: int, spec_low: PrecisionSpec,
                             kahan: bool, n_paths: int,
                             cost: Optional[CostModel] = None) -> LevelStats:
    acc = (N.Moments * 3)(m.d_hat.to_c(), m.d_bar.to_c(), m.d_four.to_c())
    out = N.LevelStatsC()
    cm = (cost or CostModel())._c()
    N.load().lpmc_level_stats_from_moments(acc, int(level), C.byref(spec_low._c()),
                                           int(bool(kahan)), C.byref(cm), int(n_paths),
                                           C.byref(out))
    return LevelStats.from_c(out)


def level_partials(model: SdeModel, level: int, spec_low: PrecisionSpec,
                   approx: Optional[InvCdfApprox], kahan: bool, n_paths: int, seed: int,
                   path_base: int, chunk_begin: int, chunk_end: int, **ext) -> np.ndarray:
    """Chunk accumulators for chunks [chunk_begin, chunk_end) as an
    (n_chunks, 3, 5) float64 array of raw states {n, mean, m2, m3, m4}."""
    k = max(int(chunk_end) - int(chunk_begin), 0)
    acc = (N.Moments * max(3 * k, 1))()
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_level_partials(C.byref(_gbm_c(model)), int(level),
                                         C.byref(spec_low._c()), _table_ptr(approx),
                                         int(bool(kahan)), int(n_paths), int(seed),
                                         int(path_base), int(chunk_begin), int(chunk_end),
                                         C.byref(opts), acc, C.byref(err)), err)
    out = np.zeros((k, 3, 5))
    for i in range(3 * k):
        out[i // 3, i % 3] = acc[i].as_tuple()
    return out


def fold_partials(parts: np.ndarray) -> CoupledMoments:
    """Index-order fold (mlmc.hpp:108-110) of (n_chunks, 3, 5) partials."""
    parts = np.asarray(parts, dtype=np.float64).reshape(-1, 3, 5)
    k = parts.shape[0]
    acc = (N.Moments * max(3 * k, 1))()
    for i in range(3 * k):
        row = parts[i // 3, i % 3]
        acc[i] = N.Moments(int(row[0]), row[1], row[2], row[3], row[4])
    out = (N.Moments * 3)()
    N.load().lpmc_fold_partials(acc, k, out)
    return CoupledMoments.from_c3(out)


def simulate_paths(model: SdeModel, level: int, spec_low: PrecisionSpec,
                   approx: Optional[InvCdfApprox], kahan: bool, n_paths: int, seed: int,
                   path_base: int, want_z: bool = False, **ext):
    """Per-path terminal values (n, 4) as simulate_coupled returns them
    (sde.hpp:279-283), computed by the device kernel; optionally the exact
    Gaussians (n, 2^level) the hat legs consumed."""
    out = np.zeros((int(n_paths), 4))
    z = np.zeros((int(n_paths), 1 << int(level))) if want_z else None
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_simulate_paths(C.byref(_gbm_c(model)), int(level),
                                         C.byref(spec_low._c()), _table_ptr(approx),
                                         int(bool(kahan)), int(n_paths), int(seed),
                                         int(path_base), C.byref(opts),
                                         out.ctypes.data_as(N._dp),
                                         z.ctypes.data_as(N._dp) if want_z else None,
                                         C.byref(err)), err)
    return (out, z) if want_z else out


def device_inv_cdf(u: np.ndarray, approx: Optional[InvCdfApprox] = None,
                   device: Optional[int] = None, exact_z: str = "fast") -> np.ndarray:
    """Exact (approx None) or approximate inverse CDF of host uniforms,
    evaluated by the kernels' device functions (exact Gaussians in the
    ``exact_z`` mode: "fast" or "glibc")."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    out = np.zeros_like(u)
    err = N.Error()
    opts = _options(device=device, exact_z=exact_z)
    N.check(N.load().lpmc_device_inv_cdf(u.ctypes.data_as(N._dp), len(u), _table_ptr(approx),
                                         out.ctypes.data_as(N._dp), C.byref(opts),
                                         C.byref(err)), err)
    return out


def device_math(op: str, x: np.ndarray, approx: Optional[InvCdfApprox] = None,
                device: Optional[int] = None) -> np.ndarray:
    """Diagnostics: op in {"exact", "approx", "exact_libdevice", "erfc",
    "exact_glibc"}."""
    ops = {"exact": 0, "approx": 1, "exact_libdevice": 2, "erfc": 3, "exact_glibc": 5}
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    err = N.Error()
    opts = _options(device=device)
    N.check(N.load().lpmc_device_math(ops[op], x.ctypes.data_as(N._dp), len(x),
                                      _table_ptr(approx), out.ctypes.data_as(N._dp),
                                      C.byref(opts), C.byref(err)), err)
    return out


def erfc_core(t: float) -> float:
    """Host evaluation of the device erfc core (bitwise the device's)."""
    return float(N.load().lpmc_erfc_core(float(t)))


def bar_arithmetic(model: SdeModel, level: int, spec_low: PrecisionSpec,
                   approx: Optional[InvCdfApprox], kahan: bool, **ext) -> dict:
    """The arithmetic a production launch of this run uses for the low-precision
    legs (lpmc_bar_arithmetic; a host decision, no device needed)."""
    out = C.c_int32(0)
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_bar_arithmetic(C.byref(_gbm_c(model)), int(level),
                                         C.byref(spec_low._c()), _table_ptr(approx),
                                         int(bool(kahan)), C.byref(opts), C.byref(out),
                                         C.byref(err)), err)
    names = ["carrier", "fp32", "fp32-round", "fp64-round", "half2-ieee"]
    return {"arith": names[out.value & 0xff], "pow2_folded": bool(out.value & 0x100),
            "native_binary16": bool(out.value & 0x200),
            "native_bfloat16": bool(out.value & 0x400)}


def phi_inv_direct_core(v: float) -> Optional[float]:
    """Host evaluation of the direct table of the default exact inverse CDF
    (bitwise the device's value) for v = min(u, 1 - u) in [2^-15, 1/2]; None
    outside the table."""
    ok = C.c_int32(0)
    z = float(N.load().lpmc_phi_inv_direct_core(float(v), C.byref(ok)))
    return z if ok.value else None


def glibc_math(op: str, x: float) -> Optional[float]:
    """Host evaluation of the restated glibc routine (op in {"exp", "log",
    "erfc", "inv_cdf"}), bitwise the device's LPMC_EXACT_Z_GLIBC path; None
    where the argument is outside the restated ranges."""
    ok = N.C.c_int32(0)
    r = float(N.load().lpmc_glibc_math({"exp": 0, "log": 1, "erfc": 2, "inv_cdf": 3}[op],
                                       float(x), N.C.byref(ok)))
    return r if ok.value else None


class LevelPlan:
    """Device-resident repeated launches of one level (buffers and table
    stay in HBM).  launch() only enqueues; collect() waits and folds."""

    def __init__(self, model: SdeModel, level: int, spec_low: PrecisionSpec,
                 approx: Optional[InvCdfApprox], kahan: bool, n_paths: int, seed: int,
                 path_base: int = 0, chunks: Optional[tuple] = None, **ext):
        self._lib = N.load()
        self._h = C.c_void_p()
        err = N.Error()
        opts = _options(**ext)
        n_chunks = (int(n_paths) + N.CHUNK_PATHS - 1) // N.CHUNK_PATHS
        c0, c1 = chunks if chunks is not None else (0, n_chunks)
        N.check(self._lib.lpmc_plan_create_range(C.byref(_gbm_c(model)), int(level),
                                                 C.byref(spec_low._c()), _table_ptr(approx),
                                                 int(bool(kahan)), int(n_paths), int(seed),
                                                 int(path_base), int(c0), int(c1),
                                                 C.byref(opts), C.byref(self._h),
                                                 C.byref(err)), err)
        self.level = level
        self.n_paths = n_paths
        self.chunks = (c0, c1)

    def collect_partials(self) -> np.ndarray:
        """(n_chunks, 3, 5) raw chunk accumulators of this plan's shard."""
        k = self.chunks[1] - self.chunks[0]
        acc = (N.Moments * (3 * k))()
        err = N.Error()
        N.check(self._lib.lpmc_plan_collect_partials(self._h, acc, C.byref(err)), err)
        out = np.zeros((k, 3, 5))
        for i in range(3 * k):
            out[i // 3, i % 3] = acc[i].as_tuple()
        return out

    def launch(self, stream: Optional[int] = None) -> None:
        err = N.Error()
        N.check(self._lib.lpmc_plan_launch(self._h, None if stream is None else int(stream),
                                           C.byref(err)), err)

    def collect(self) -> CoupledMoments:
        acc = (N.Moments * 3)()
        err = N.Error()
        N.check(self._lib.lpmc_plan_collect(self._h, acc, C.byref(err)), err)
        return CoupledMoments.from_c3(acc)

    def kernels_per_launch(self) -> int:
        return int(self._lib.lpmc_plan_kernels_per_launch(self._h))

    def close(self) -> None:
        if self._h:
            self._lib.lpmc_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def measure_pipe_peaks(device: Optional[int] = None) -> dict:
    """Measured lane-op rates (ops/s) of the device: fp64 / fp32 / fp16 FMA
    and 64-bit integer multiply-add (the RNG's operation)."""
    out = np.zeros(4)
    err = N.Error()
    N.check(N.load().lpmc_measure_pipe_peaks(-1 if device is None else int(device),
                                             out.ctypes.data_as(N._dp), C.byref(err)), err)
    return {"fp64_ops_per_s": out[0], "fp32_ops_per_s": out[1], "fp16_ops_per_s": out[2],
            "mul64_ops_per_s": out[3]}


def device_count() -> int:
    return int(N.load().lpmc_device_count())


def launch_count() -> int:
    return int(N.load().lpmc_launch_count())


def reset_launch_count() -> None:
    N.load().lpmc_reset_launch_count()


# -------------------------------------- estimator layer (mlmc.hpp:151-285) --
class AllocationKind:
    standard = N.ALLOCATION_STANDARD
    nested = N.ALLOCATION_NESTED


@dataclass
class Allocation:
    """mlmc.hpp:153-163."""
    primary: list = field(default_factory=list)
    secondary: list = field(default_factory=list)
    degenerate: bool = False


@dataclass
class PredictedTimes:
    t_hat: float = 0.0
    t_bar: float = 0.0


@dataclass
class SpeedupResult:
    value: float = 0.0
    cost_ratio_only: bool = False


@dataclass
class EstimatorResult:
    """mlmc.hpp:232-239."""
    value: float = 0.0
    level_contributions: list = field(default_factory=list)
    pilot_stats: list = field(default_factory=list)
    allocation: Allocation = field(default_factory=Allocation)
    times: PredictedTimes = field(default_factory=PredictedTimes)
    eps: float = 0.0


def _stats_array(stats):
    stats = list(stats)
    arr = (N.LevelStatsC * max(1, len(stats)))()
    for i, s in enumerate(stats):
        arr[i] = s._c()
    return arr, len(stats)


def allocate_samples(stats, eps: float, kind: int) -> Allocation:
    """allocate_samples (mlmc.hpp:165-195), bitwise (host C++)."""
    arr, n = _stats_array(stats)
    prim = (C.c_uint64 * max(1, n))()
    sec = (C.c_uint64 * max(1, n))()
    deg = C.c_int32()
    err = N.Error()
    N.check(N.load().lpmc_allocate_samples(arr, n, float(eps), int(kind), prim, sec,
                                           C.byref(deg), C.byref(err)), err)
    return Allocation([int(x) for x in prim[:n]],
                      [int(x) for x in sec[:n]] if kind == AllocationKind.nested else [],
                      bool(deg.value))


def predicted_times(stats, eps: float) -> PredictedTimes:
    """predicted_times (mlmc.hpp:202-213), bitwise (host C++)."""
    arr, n = _stats_array(stats)
    th, tb = C.c_double(), C.c_double()
    err = N.Error()
    N.check(N.load().lpmc_predicted_times(arr, n, float(eps), C.byref(th), C.byref(tb),
                                          C.byref(err)), err)
    return PredictedTimes(th.value, tb.value)


def per_level_speedup(s: LevelStats) -> SpeedupResult:
    """per_level_speedup (mlmc.hpp:223-230), bitwise (host C++)."""
    v = C.c_double()
    flag = C.c_int32()
    err = N.Error()
    N.check(N.load().lpmc_per_level_speedup(C.byref(s._c()), C.byref(v), C.byref(flag),
                                            C.byref(err)), err)
    return SpeedupResult(v.value, bool(flag.value))


def run_nested_estimator(model: SdeModel, max_level: int, spec_low: PrecisionSpec,
                         approx: Optional[InvCdfApprox], kahan: bool, eps: float, seed: int,
                         cost: Optional[CostModel] = None, threads: int = 1,
                         pilot_paths: int = 1000, **ext) -> EstimatorResult:
    """run_nested_estimator (mlmc.hpp:244-283) on the device: the pilot pass
    and the main pass each run all their levels concurrently."""
    if max_level < 0:
        raise InvalidArgument("max level must be >= 0")
    L = int(max_level) + 1
    contrib = (C.c_double * L)()
    pilot = (N.LevelStatsC * L)()
    prim = (C.c_uint64 * L)()
    sec = (C.c_uint64 * L)()
    res = N.EstimatorResultC()
    res.level_contributions = C.cast(contrib, N._dp)
    res.pilot_stats = C.cast(pilot, C.POINTER(N.LevelStatsC))
    res.primary = C.cast(prim, C.POINTER(C.c_uint64))
    res.secondary = C.cast(sec, C.POINTER(C.c_uint64))
    err = N.Error()
    opts = _options(**ext)
    cm = (cost or CostModel())._c()
    N.check(N.load().lpmc_run_nested_estimator(C.byref(_gbm_c(model)), int(max_level),
                                               C.byref(spec_low._c()), _table_ptr(approx),
                                               int(bool(kahan)), float(eps), int(seed),
                                               C.byref(cm), int(pilot_paths), C.byref(opts),
                                               C.byref(res), C.byref(err)), err)
    return EstimatorResult(
        value=res.value, level_contributions=list(contrib),
        pilot_stats=[LevelStats.from_c(pilot[i]) for i in range(L)],
        allocation=Allocation([int(x) for x in prim], [int(x) for x in sec],
                              bool(res.degenerate)),
        times=PredictedTimes(res.t_hat, res.t_bar), eps=res.eps)


# ---------------------------------------- step-error probe (sde.hpp:289-344) --
@dataclass
class StepErrorStats:
    mean_eta: float = 0.0
    mean_abs_eta: float = 0.0
    mean_eta_prime: float = 0.0
    mean_abs_eta_prime: float = 0.0
    samples: int = 0


def step_error_probe(model: SdeModel, level: int, spec: PrecisionSpec,
                     approx: Optional[InvCdfApprox], n_samples: int, seed: int,
                     **ext) -> StepErrorStats:
    """step_error_probe (sde.hpp:297-344) on the device: eta / eta' residual
    means over n_samples steps of the paths 0, 1, ... of ``seed``."""
    out = N.StepErrorStatsC()
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_step_error_probe(C.byref(_gbm_c(model)), int(level), C.byref(spec._c()),
                                           _table_ptr(approx), int(n_samples), int(seed),
                                           C.byref(opts), C.byref(out), C.byref(err)), err)
    return StepErrorStats(out.mean_eta, out.mean_abs_eta, out.mean_eta_prime,
                          out.mean_abs_eta_prime, int(out.samples))


# ---------------------------------- density histogram (experiments.hpp:276) --
def density_histogram(approx: Optional[InvCdfApprox], seed: int, n_samples: int, z_max: float,
                      bin_width: float, n_bins: int, **ext) -> np.ndarray:
    """Counts of run_density_report's histogram (experiments.hpp:276-285) on
    the device: draws 0..n-1 of UniformStream(seed, 0) through the table
    (None = exact inverse CDF), bin (int)((z + z_max) / bin_width) clamped."""
    bins = np.zeros(int(n_bins), dtype=np.uint64)
    err = N.Error()
    opts = _options(**ext)
    N.check(N.load().lpmc_density_histogram(_table_ptr(approx), int(seed), int(n_samples),
                                            float(z_max), float(bin_width), int(n_bins),
                                            bins.ctypes.data_as(C.POINTER(C.c_uint64)),
                                            C.byref(opts), C.byref(err)), err)
    return bins
