"""Experiment drivers above the level sampler: the Python mirror of the
reference's experiments.hpp (proj/include/lpmc/experiments.hpp:22-246).

==========================  ================================================
this module                 reference
==========================  ================================================
ExperimentConfig            experiments.hpp:22-75
TwoWayRow /                 experiments.hpp:79-151 (simulate_two_way per
run_two_way_experiment        path, run_batched merge)
FourWayRow / FourWayOutput  experiments.hpp:154-216 (three estimate_level_stats
run_four_way_experiment       per level: low, low+Kahan, high)
SpeedupRow /                experiments.hpp:218-246 (per_level_speedup)
run_speedup_report
StepErrorRow /              experiments.hpp:297-319 (device step_error_probe)
run_step_error_report
DensityRow /                experiments.hpp:252-295 (device histogram and curve)
run_density_report
==========================  ================================================

Same path bases, path counts and merge order as the reference, so every row
is the reference's row up to the device's exact-Gaussian ulps (bitwise for
table-driven bar legs with ``reduce="sequential"``).  The B200 difference is
the schedule: all (precision, level) runs of an experiment are handed to the
device at once (``run_coupled_many``), so the small levels run concurrently
instead of one after another.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

import math

import numpy as np

from .api import (CostModel, InvalidArgument, InvCdfApprox, LevelStats, PrecisionSpec,
                  StepErrorStats, density_histogram, device_inv_cdf, level_stats_from_moments,
                  make_gbm, per_level_speedup, run_coupled_many, step_error_probe)


@dataclass
class ExperimentConfig:
    mu: float = 0.05
    sigma: float = 0.2
    x0: float = 1.0
    horizon: float = 1.0
    precisions: List[str] = field(default_factory=lambda: ["fp16"])
    approx: str = "linear:1024"
    kahan: bool = False
    level_min: int = 0
    level_max: int = 12
    paths: List[int] = field(default_factory=list)
    seed: int = 1
    cost: CostModel = field(default_factory=CostModel)
    threads: int = 1  # scheduled the CPU reference only; accepted and ignored

    def model(self):
        return make_gbm(self.mu, self.sigma, self.x0, self.horizon)

    def paths_for_level(self, level: int) -> int:
        """experiments.hpp:45-54."""
        if self.paths:
            idx = 0 if len(self.paths) == 1 else level - self.level_min
            if idx >= len(self.paths):
                raise InvalidArgument("paths list shorter than level range")
            return int(self.paths[idx])
        if level <= 9:
            return 10000
        return max(2, 10000 >> (level - 9))

    def validate(self) -> None:
        """experiments.hpp:56-66."""
        if self.level_min < 0 or self.level_max < self.level_min:
            raise InvalidArgument("empty or negative level range")
        if not self.precisions:
            raise InvalidArgument("no precision given")
        for p in self.precisions:
            PrecisionSpec.parse(p)
        if self.approx != "exact":
            InvCdfApprox.parse(self.approx)
        for level in range(self.level_min, self.level_max + 1):
            if self.paths_for_level(level) < 2:
                raise InvalidArgument("need at least 2 paths per level")

    def build_approx(self) -> Optional[InvCdfApprox]:
        return None if self.approx == "exact" else InvCdfApprox.parse(self.approx)


@dataclass
class TwoWayRow:
    n_steps: int
    precision: str
    kahan: bool
    variance: float
    stderr_variance: float
    paths: int


def run_two_way_experiment(config: ExperimentConfig, **ext) -> List[TwoWayRow]:
    """experiments.hpp:119-151: Var(X_hat_N - X_bar_N) per (precision, level),
    path base (pi << 48) | (l << 40)."""
    config.validate()
    approx = config.build_approx()
    runs, keys = [], []
    for pi, name in enumerate(config.precisions):
        spec = PrecisionSpec.parse(name)
        for level in range(config.level_min, config.level_max + 1):
            n = config.paths_for_level(level)
            runs.append((level, spec, config.kahan, n, (pi << 48) | (level << 40)))
            keys.append((name, level, n))
    ext = dict(ext)
    ext["legs"] = "fine"
    res = run_coupled_many(config.model(), approx, config.seed, runs, **ext)
    rows = []
    for (name, level, n), m in zip(keys, res):
        acc = m.d_four  # x_hat - x_bar
        rows.append(TwoWayRow(1 << level, name, bool(config.kahan), acc.variance(),
                              acc.variance_stderr(), n))
    return rows


@dataclass
class FourWayRow:
    level: int
    series: str
    variance: float
    stderr_variance: float
    paths: int


@dataclass
class FourWayOutput:
    rows: List[FourWayRow] = field(default_factory=list)
    low_stats: List[LevelStats] = field(default_factory=list)
    low_kahan_stats: List[LevelStats] = field(default_factory=list)
    high_stats: List[LevelStats] = field(default_factory=list)


def run_four_way_experiment(config: ExperimentConfig, **ext) -> FourWayOutput:
    """experiments.hpp:170-216: per level the low, low+Kahan and high
    estimate_level_stats (path bases l << 40 | {0, 1, 2} << 36), six series."""
    config.validate()
    approx = config.build_approx()
    low_name = config.precisions[0]
    high_name = config.precisions[1] if len(config.precisions) > 1 else "fp32"
    low, high = PrecisionSpec.parse(low_name), PrecisionSpec.parse(high_name)
    runs, meta = [], []
    for level in range(config.level_min, config.level_max + 1):
        n = config.paths_for_level(level)
        base = level << 40
        for spec, kahan, phase in ((low, False, 0), (low, True, 1), (high, False, 2)):
            runs.append((level, spec, kahan, n, base | (phase << 36)))
            meta.append((level, spec, kahan, n))
    res = run_coupled_many(config.model(), approx, config.seed, runs, **ext)
    stats = [level_stats_from_moments(m, level, spec, kahan, n, config.cost)
             for m, (level, spec, kahan, n) in zip(res, meta)]
    out = FourWayOutput()
    for i, level in enumerate(range(config.level_min, config.level_max + 1)):
        s0, s1, s2 = stats[3 * i:3 * i + 3]
        n = config.paths_for_level(level)
        out.low_stats.append(s0)
        out.low_kahan_stats.append(s1)
        out.high_stats.append(s2)
        out.rows += [FourWayRow(level, "two_way_exact", s0.v_hat, s0.v_hat_stderr, n),
                     FourWayRow(level, "two_way_" + low_name, s0.v_bar, s0.v_bar_stderr, n),
                     FourWayRow(level, "two_way_" + low_name + "_kahan", s1.v_bar,
                                s1.v_bar_stderr, n),
                     FourWayRow(level, "four_way_" + high_name, s2.V_bar, s2.V_bar_stderr, n),
                     FourWayRow(level, "four_way_" + low_name, s0.V_bar, s0.V_bar_stderr, n),
                     FourWayRow(level, "four_way_" + low_name + "_kahan", s1.V_bar,
                                s1.V_bar_stderr, n)]
    return out


@dataclass
class SpeedupRow:
    level: int
    variant: str
    speedup: float
    cost_ratio_only: bool


def run_speedup_report(high_stats, low_stats, low_kahan_stats) -> List[SpeedupRow]:
    """experiments.hpp:225-246."""
    if not high_stats:
        raise InvalidArgument("missing level stats")
    rows = []
    for i, hs in enumerate(high_stats):
        r = per_level_speedup(hs)
        rows.append(SpeedupRow(hs.level, "single", r.value, r.cost_ratio_only))
        if i < len(low_stats):
            r = per_level_speedup(low_stats[i])
            rows.append(SpeedupRow(low_stats[i].level, "half", r.value, r.cost_ratio_only))
        if i < len(low_kahan_stats):
            r = per_level_speedup(low_kahan_stats[i])
            rows.append(SpeedupRow(low_kahan_stats[i].level, "half_kahan", r.value,
                                   r.cost_ratio_only))
    return rows


@dataclass
class StepErrorRow:
    level: int
    stats: StepErrorStats


def run_step_error_report(config: ExperimentConfig, samples: int, **ext) -> List[StepErrorRow]:
    """experiments.hpp:302-319."""
    config.validate()
    if samples < 10000:
        raise InvalidArgument("step-error probe needs >= 1e4 samples")
    approx = config.build_approx()
    spec = PrecisionSpec.parse(config.precisions[0])
    model = config.model()
    return [StepErrorRow(level, step_error_probe(model, level, spec, approx, samples, config.seed,
                                                 **ext))
            for level in range(config.level_min, config.level_max + 1)]


@dataclass
class DensityRow:
    series: str  # "curve" or "hist"
    x: float
    y: float


def run_density_report(config: ExperimentConfig, curve_points: int = 2048,
                       hist_samples: int = 1000000, bin_width: float = 0.05,
                       **ext) -> List[DensityRow]:
    """experiments.hpp:258-295: the inverse-CDF curve at u = i / curve_points
    and the histogram of hist_samples draws of UniformStream(seed, 0), both
    evaluated on the device; bin geometry and densities as the reference."""
    config.validate()
    approx = config.build_approx()
    u = np.arange(1, curve_points, dtype=np.float64) / curve_points
    dev = ext.get("device")
    zmode = ext.get("exact_z", "fast")
    curve = device_inv_cdf(u, approx, device=dev, exact_z=zmode) if len(u) else np.zeros(0)
    rows = [DensityRow("curve", float(a), float(b)) for a, b in zip(u, curve)]
    if approx is not None:
        z_max = approx.max_value()
    else:
        z_max = float(device_inv_cdf(np.array([1.0 - 2.0 ** -30]), None, device=dev,
                                     exact_z=zmode)[0])
    n_bins = int(math.ceil(2.0 * z_max / bin_width)) + 1
    bins = density_histogram(approx, config.seed, hist_samples, z_max, bin_width, n_bins, **ext)
    for b in range(n_bins):
        center = -z_max + (b + 0.5) * bin_width
        rows.append(DensityRow("hist", center, float(bins[b]) / (float(hist_samples) * bin_width)))
    return rows
