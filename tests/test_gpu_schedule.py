"""The warp-per-path schedule (wpp_kernel, LPMC_SCHEDULE_WARP_PER_PATH) against
the fused level kernel: same draws, same step functions, same batch tree, so
every per-path value and every moment is bitwise the same -- and, in glibc
mode, bitwise the reference's (golden vectors)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits, unhex

pytestmark = pytest.mark.gpu

W = {"schedule": "warp_per_path"}
F = {"schedule": "fused"}


def _state(m):
    return [m.d_hat.state(), m.d_bar.state(), m.d_four.state()]


CASES = [  # level, mantissa bits, approx, kahan, legs, payoff
    (1, 23, "linear:16", False, "all", "terminal"),
    (2, 10, "linear:16", True, "all", "terminal"),
    (4, 23, "exact", True, "all", "call"),
    (5, 52, "exact", False, "hat", "terminal"),
    (6, 10, "constant:16", False, "bar", "terminal"),
    (6, 16, "cubic:64", True, "all", "terminal"),
    (7, 23, "linear:1024", False, "fine", "terminal"),
    (9, 7, "linear:16", True, "all", "call"),
    (10, 23, "linear:16", False, "all", "terminal"),
]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("reduce", ["tree", "sequential"])
def test_wpp_moments_equal_fused(gpu, case, reduce):
    level, m, approx, kahan, legs, payoff = case
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    args = (gpu.make_gbm(), level, gpu.PrecisionSpec(m), tb, kahan, 3001, 7, level << 40)
    ext = dict(legs=legs, payoff=payoff, reduce=reduce)
    assert _state(gpu.run_coupled_paths(*args, **ext, **W)) == \
           _state(gpu.run_coupled_paths(*args, **ext, **F))


@pytest.mark.parametrize("case", CASES)
def test_wpp_paths_equal_fused(gpu, case):
    level, m, approx, kahan, legs, payoff = case
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    args = (gpu.make_gbm(), level, gpu.PrecisionSpec(m), tb, kahan, 517, 3, 5)
    a = gpu.simulate_paths(*args, legs=legs, **W)
    b = gpu.simulate_paths(*args, legs=legs, **F)
    assert np.array_equal(bits(a), bits(b))


@pytest.mark.parametrize("idx", range(0, 165, 4))
def test_wpp_glibc_paths_golden(gpu, golden, idx):
    """Warp-per-path in glibc mode: all four legs bitwise the reference's."""
    c = golden["paths"][idx]
    if c["level"] == 0:
        pytest.skip("level 0 runs fused")
    want = unhex(c["out"]).reshape(-1, 4)
    tb = None if c["approx"] == "exact" else gpu.InvCdfApprox.parse(c["approx"])
    out = gpu.simulate_paths(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]), tb,
                             bool(c["kahan"]), want.shape[0], c["seed"], c["path_base"],
                             exact_z="glibc", **W)
    assert np.array_equal(bits(out), bits(want))


def test_wpp_failures_and_range_fallback(gpu):
    P = gpu.PrecisionSpec
    bad = gpu.make_gbm(1e30, 0.0, 1e300)
    errs = []
    for ext in (W, F):
        with pytest.raises(gpu.DomainError, match="non-finite operand") as ei:
            gpu.run_coupled_paths(bad, 4, P.carrier(), None, False, 600, 1, 0, **ext)
        errs.append((ei.value.path_index, ei.value.step))
    assert errs[0] == errs[1]
    hot = gpu.make_gbm(80.0, 0.2)  # native fp32 legs leave the exact range: emulated re-run
    tb = gpu.InvCdfApprox.parse("linear:16")
    args = (hot, 4, P.fp32(), tb, True, 1000, 2, 0)
    assert _state(gpu.run_coupled_paths(*args, **W)) == _state(gpu.run_coupled_paths(*args, **F))


def test_auto_schedule_callers_unchanged(gpu):
    """The two-way experiment and the nested estimator (small deep runs: the
    auto schedule picks warp-per-path) give the fused schedule's numbers."""
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_two_way_experiment
    cfg = ExperimentConfig(precisions=["fp16"], approx="linear:64", level_min=0, level_max=11,
                           paths=[2000])
    a = run_two_way_experiment(cfg, reduce="sequential")
    b = run_two_way_experiment(cfg, reduce="sequential", **F)
    assert [(r.variance, r.stderr_variance) for r in a] == [(r.variance, r.stderr_variance) for r in b]
    tb = gpu.InvCdfApprox.parse("linear:16")
    r1 = gpu.run_nested_estimator(gpu.make_gbm(), 6, gpu.PrecisionSpec.fp16(), tb, False, 2e-3, 1)
    r2 = gpu.run_nested_estimator(gpu.make_gbm(), 6, gpu.PrecisionSpec.fp16(), tb, False, 2e-3, 1, **F)
    assert r1.value == r2.value and r1.level_contributions == r2.level_contributions
