"""The reference's acceptance gate (proj/tests/acceptance.cpp:86-257, criteria
SPEC.md:466-474) re-hosted on the device: the same configurations, seeds and
thresholds, every quantity computed by the sampler through the public API.
Criterion 1 (softfloat grid oracle) is host arithmetic, pinned bitwise in
tests/test_oracle.py; criterion 9 is the CLI (out of scope).  Each criterion
runs in the fast mode (default) and with exact_z="glibc", where the numbers
are the reference's own bit for bit.  The same gate at 10x the reference's
path counts closes out the file (GPU scale).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MODES = [{}, {"exact_z": "glibc"}]


def slope(xs, ys):
    """acceptance.cpp:31-47 (least squares)."""
    mx = sum(xs) / len(xs)
    my = sum(ys) / len(ys)
    sxy = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    sxx = sum((x - mx) ** 2 for x in xs)
    return sxy / sxx


@pytest.mark.parametrize("ext", MODES)
def test_c2_zero_mean_rounding_signature(gpu, ext):
    """acceptance.cpp:106-114: fp16 step residuals have zero mean."""
    s = gpu.step_error_probe(gpu.make_gbm(), 8, gpu.PrecisionSpec.fp16(), None, 1000000, 2, **ext)
    assert abs(s.mean_eta) <= 0.05 * s.mean_abs_eta, (s.mean_eta, s.mean_abs_eta)


def _two_way(kahan, paths, **ext):
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_two_way_experiment
    cfg = ExperimentConfig(precisions=["fp16", "bf16"], approx="cubic:64", kahan=kahan,
                           level_min=4, level_max=12, paths=[paths], seed=1)
    return run_two_way_experiment(cfg, **ext)


def _rows_slope(rows, lo, hi):
    return slope([math.log2(r.n_steps) for r in rows[lo:hi]],
                 [math.log2(r.variance) for r in rows[lo:hi]])


def _check_c3_c4(gpu, paths, ext):
    plain = _two_way(False, paths, **ext)
    s3 = _rows_slope(plain, 0, 9)  # fp16 rows first
    assert 0.7 <= s3 <= 1.6, s3                                # criterion 3
    kahan = _two_way(True, paths, **ext)
    s4 = _rows_slope(kahan, 0, 9)
    ratio = sum(kahan[9 + i].variance / kahan[i].variance for i in range(9)) / 9.0
    assert abs(s4) <= 0.3 and 16.0 <= ratio <= 256.0, (s4, ratio)  # criterion 4
    return s3, s4, ratio


@pytest.mark.parametrize("ext", MODES)
def test_c3_c4_two_way_growth_and_kahan_flattening(gpu, ext):
    """acceptance.cpp:118-166."""
    print(_check_c3_c4(gpu, 10000, ext))


def _crossover(stats):
    """acceptance.cpp:174-178."""
    for s in stats:
        if s.V_bar >= 0.25 * s.v_bar:
            return s.level
    return stats[-1].level + 1


def _check_c5_c6_c7(gpu, paths, ext):
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_four_way_experiment
    cfg = ExperimentConfig(precisions=["fp16", "fp32"], approx="linear:32", level_min=0,
                           level_max=12, paths=[paths], seed=1)
    out = run_four_way_experiment(cfg, **ext)
    cross_plain = _crossover(out.low_stats)
    cross_kahan = _crossover(out.low_kahan_stats)
    drops = [out.low_stats[l].V_bar / out.low_stats[l].v_hat for l in range(5)]
    assert 6 <= cross_plain <= 8 and 9 <= cross_kahan <= 12, (cross_plain, cross_kahan)
    assert max(drops) <= 2.0 ** -5 and drops[0] <= 2.0 ** -8, drops            # criterion 5
    s6 = slope([-float(l) for l in range(2, 13)],
               [math.log2(out.high_stats[l].V_bar) for l in range(2, 13)])
    assert 0.7 <= s6 <= 1.3, s6                                                 # criterion 6
    single = [gpu.per_level_speedup(out.high_stats[l]).value for l in range(4, 11)]
    half = [gpu.per_level_speedup(out.low_stats[l]).value for l in range(0, 3)]
    assert all(4.5 <= s <= 7.0 for s in single) and all(8.0 <= s <= 14.0 for s in half), \
        (single, half)                                                          # criterion 7
    return cross_plain, cross_kahan, s6


@pytest.mark.parametrize("ext", MODES)
def test_c5_c6_c7_four_way(gpu, ext):
    """acceptance.cpp:180-243: crossovers, fp32 decay, per-level speedups."""
    print(_check_c5_c6_c7(gpu, 10000, ext))


@pytest.mark.parametrize("ext", MODES)
def test_c8_estimator_correctness(gpu, ext):
    """acceptance.cpp:247-277."""
    P = gpu.PrecisionSpec
    det = gpu.make_gbm(0.05, 0.0)
    r_det = gpu.run_nested_estimator(det, 4, P.carrier(), None, False, 0.01, 1, **ext)
    expected = (1.0 + 0.05 * 2.0 ** -4) ** 16.0
    assert abs(r_det.value - expected) <= 8.0 * np.finfo(float).eps * expected
    r_car = gpu.run_nested_estimator(gpu.make_gbm(), 3, P.carrier(), None, False, 0.05, 1, **ext)
    assert all(s.V_bar == 0.0 for s in r_car.pilot_stats)
    eps = 1e-3
    r = gpu.run_nested_estimator(gpu.make_gbm(), 8, P.fp32(), gpu.InvCdfApprox.parse("linear:1024"),
                                 False, eps, 1, **ext)
    bias = math.exp(0.05) - (1.0 + 0.05 / 256.0) ** 256.0
    assert abs(r.value - math.exp(0.05)) <= 3.0 * eps + abs(bias)


def test_gate_at_gpu_scale(gpu):
    """Criteria 3-7 at 10x the reference's 1e4 paths per level (the gate is
    statistical; more paths tighten every slope and ratio)."""
    print(_check_c3_c4(gpu, 100000, {}), _check_c5_c6_c7(gpu, 100000, {}))
