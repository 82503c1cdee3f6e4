"""GPU parity of the callers above the level sampler:
the two-way sampler (simulate_two_way, sde.hpp:162-196) and experiment
(experiments.hpp:119-151), the concurrent multi-run entry point, and the
nested estimator (mlmc.hpp:244-283), against fixtures from the unmodified
reference (tests/golden/callers_vectors.json) and the C oracle.

Contract: as test_gpu_parity.py -- table-driven bar legs bitwise, all legs
bitwise given the device's own exact Gaussians (oracle replay), carrier legs
within libm tolerance of glibc; allocation counts equal; estimator
contributions within 1e-12 absolute (means of O(1e-3)-variance differences).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import ROOT, bits, unhex

pytestmark = pytest.mark.gpu

CALLERS = os.path.join(ROOT, "tests", "golden", "callers_vectors.json")


@pytest.fixture(scope="module")
def cv():
    with open(CALLERS) as f:
        return json.load(f)


def _table(lib, name):
    return None if name == "exact" else lib.InvCdfApprox.parse(name)


@pytest.mark.parametrize("idx", range(0, 72))
def test_two_way_paths_vs_reference(gpu, cv, oracle, idx):
    cases = cv["two_way_paths"]
    if idx >= len(cases):
        pytest.skip("fewer cases")
    c = cases[idx]
    want = unhex(c["out"]).reshape(-1, 2)
    n = want.shape[0]
    out, z = gpu.simulate_paths(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                                _table(gpu, c["approx"]), bool(c["kahan"]), n, c["seed"],
                                c["path_base"], want_z=True, legs="fine")
    assert not out[:, [1, 3]].any()  # no coarse legs
    # the two-way legs are the coupled sampler's fine legs: bitwise == the
    # oracle's coupled replay on the device's own Gaussians
    cfg = oracle.config(level=c["level"], mantissa_bits=c["m"], approx=c["approx"],
                        kahan=c["kahan"], seed=c["seed"])
    rep, _, fails = oracle.simulate(cfg, c["path_base"], n, z_in=z)
    assert not fails
    assert np.array_equal(bits(out[:, [0, 2]]), bits(rep[:, [0, 2]]))
    if c["approx"] != "exact":
        assert np.array_equal(bits(out[:, 2]), bits(want[:, 1]))
    np.testing.assert_allclose(out[:, 0], want[:, 0], rtol=1e-12, atol=1e-300)


def test_two_way_moments_sequential_bitwise(gpu, oracle):
    """lpmc_run_two_way_paths (sequential order) == the reference's
    run_batched merge of x_hat - x_bar over the device's own paths."""
    model = gpu.make_gbm()
    sp, tb = gpu.PrecisionSpec.fp16(), gpu.InvCdfApprox.parse("linear:16")
    for level, n, base in [(0, 700, 5), (4, 2049, 1 << 40), (7, 513, 123)]:
        out = gpu.simulate_paths(model, level, sp, tb, True, n, 9, base, legs="fine")
        m = gpu.run_two_way_paths(model, level, sp, tb, True, n, 9, base, reduce="sequential")
        want = oracle.sequential_from_values(out[:, 0] - out[:, 2], np.zeros(n))
        assert m.state() == tuple(want[0])


def test_two_way_experiment_vs_reference(gpu, cv):
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_two_way_experiment
    for row in cv["two_way_rows"]:
        cfg = ExperimentConfig(precisions=[row["precision"]], approx=row["approx"],
                               kahan=bool(row["kahan"]), level_min=row["level_min"],
                               level_max=row["level_max"], paths=[row["paths"]])
        got = run_two_way_experiment(cfg, reduce="sequential")
        want = [unhex(r) for r in row["rows"]]
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert g.n_steps == int(w[0]) and g.paths == int(w[3])
            # x_hat carries the device's exact Gaussians: libm-level deviations
            np.testing.assert_allclose([g.variance, g.stderr_variance], w[1:3], rtol=1e-8)


def test_run_coupled_many_equals_separate_calls(gpu):
    model = gpu.make_gbm()
    P = gpu.PrecisionSpec
    tb = gpu.InvCdfApprox.parse("linear:16")
    runs = []
    for i in range(21):  # > 16 streams: slots are reused in order
        level = i % 7
        spec = [P.fp32(), P.fp16(), P.bf16(), P.carrier()][i % 4]
        runs.append((level, spec, bool(i % 2), [3000, 1, 0, 70000, 256][i % 5], (i << 36) + 17))
    many = gpu.run_coupled_many(model, tb, 5, runs)
    for (level, spec, kahan, n, base), m in zip(runs, many):
        one = gpu.run_coupled_paths(model, level, spec, tb, kahan, n, 5, base)
        assert [m.d_hat.state(), m.d_bar.state(), m.d_four.state()] == \
               [one.d_hat.state(), one.d_bar.state(), one.d_four.state()]


def test_run_coupled_many_error_order(gpu):
    model = gpu.make_gbm()
    P = gpu.PrecisionSpec
    car = P.carrier()
    with pytest.raises(gpu.InvalidArgument, match="level must be >= 0"):
        gpu.run_coupled_many(model, None, 1, [(2, car, False, 10, 0), (-1, car, False, 4, 0)])
    # n = 0 runs are skipped without validation, as run_coupled_paths does
    assert gpu.run_coupled_many(model, None, 1, [(-1, car, False, 0, 0)])[0].d_hat.count() == 0
    bad = gpu.make_gbm(1e30, 0.0, 1e300)
    with pytest.raises(gpu.DomainError) as ei:
        gpu.run_coupled_many(bad, None, 1, [(3, car, False, 0, 5), (3, car, False, 8, 200),
                                            (3, car, False, 8, 100)])
    assert ei.value.path_index == 200  # the first failing run in list order


@pytest.mark.parametrize("idx", range(4))
def test_nested_estimator_vs_reference(gpu, cv, idx):
    n = cv["nested"][idx]
    r = gpu.run_nested_estimator(gpu.make_gbm(), n["max_level"], gpu.PrecisionSpec(n["m"]),
                                 _table(gpu, n["approx"]), bool(n["kahan"]),
                                 float.fromhex(n["eps"]), n["seed"],
                                 pilot_paths=n["pilot_paths"], reduce="sequential")
    assert r.allocation.primary == n["primary"]
    assert r.allocation.secondary == n["secondary"]
    assert r.allocation.degenerate == n["degenerate"]
    pilot = unhex(n["pilot"]).reshape(-1, 16)
    for s, w in zip(r.pilot_stats, pilot):
        got = [s.mean_hat, s.v_hat, s.v_hat_stderr, s.mean_bar, s.v_bar, s.v_bar_stderr,
               s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat, s.c_bar, s.C_bar, s.m_hat,
               s.m_bar, s.M_bar, s.level]
        np.testing.assert_array_equal(got[9:], w[9:])
        if n["approx"] != "exact":  # bar legs bitwise, sequential order
            assert [s.mean_bar, s.v_bar, s.v_bar_stderr] == list(w[3:6])
        np.testing.assert_allclose(got[:9], w[:9], rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(r.level_contributions, unhex(n["contributions"]), rtol=0,
                               atol=1e-12)
    assert abs(r.value - float.fromhex(n["value"])) <= 1e-12
    np.testing.assert_allclose([r.times.t_hat, r.times.t_bar],
                               [float.fromhex(n["t_hat"]), float.fromhex(n["t_bar"])], rtol=1e-9)


def test_nested_estimator_errors(gpu, cv):
    for e in cv["nested_errors"]:
        with pytest.raises(gpu.InvalidArgument, match=e["msg"]):
            gpu.run_nested_estimator(gpu.make_gbm(), e["max_level"], gpu.PrecisionSpec.fp16(),
                                     gpu.InvCdfApprox.parse("linear:16"), False,
                                     float.fromhex(e["eps"]), 1, pilot_paths=e["pilot_paths"])


def test_four_way_experiment_matches_level_stats(gpu):
    """run_four_way_experiment (concurrent) == its definition as three
    estimate_level_stats calls per level (experiments.hpp:185-194)."""
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_four_way_experiment
    cfg = ExperimentConfig(precisions=["fp16", "fp32"], approx="linear:16", level_min=0,
                           level_max=5, paths=[3000])
    out = run_four_way_experiment(cfg)
    assert len(out.rows) == 6 * 6
    P = gpu.PrecisionSpec
    tb = gpu.InvCdfApprox.parse("linear:16")
    for i, level in enumerate(range(0, 6)):
        for got, spec, kahan, phase in ((out.low_stats[i], P.fp16(), False, 0),
                                        (out.low_kahan_stats[i], P.fp16(), True, 1),
                                        (out.high_stats[i], P.fp32(), False, 2)):
            want = gpu.estimate_level_stats(gpu.make_gbm(), level, spec, tb, kahan, 3000, 1,
                                            path_base=(level << 40) | (phase << 36))
            assert got == want


def test_cpp_api_device_part(gpu):
    """tests/cpp/api_smoke.cpp (reference-shaped C++ unit tests, incl. the
    nested-estimator pins test_mlmc.cpp:204-236) on the device."""
    import subprocess
    import tempfile
    from paper_2012_09739_b200 import _native as N
    src = os.path.join(ROOT, "tests", "cpp", "api_smoke.cpp")
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "api_smoke")
        subprocess.check_call(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src,
                               "-o", exe, "-L", os.path.dirname(N.LIB_PATH), "-llpmc_b200",
                               "-Wl,-rpath," + os.path.dirname(N.LIB_PATH)])
        out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stdout + out.stderr
        assert "device ok" in out.stdout


# ------------------------------------------------ step_error_probe (row 3) --
EPS = 2.0 ** -52


@pytest.mark.parametrize("idx", range(8))
def test_step_error_probe_vs_reference(gpu, cv, idx):
    c = cv["step_error"][idx]
    want = unhex(c["out"])
    r = gpu.step_error_probe(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                             _table(gpu, c["approx"]), c["n_samples"], c["seed"])
    got = np.array([r.mean_eta, r.mean_abs_eta, r.mean_eta_prime, r.mean_abs_eta_prime,
                    r.samples], dtype=np.float64)
    n = c["n_samples"]
    if n == 0:  # 0 / 0, as the reference
        assert np.all(np.isnan(got[:4])) and r.samples == 0
        return
    assert r.samples == n
    if c["approx"] != "exact":
        # identical residuals, different summation order: both sums are within
        # n eps sum|r| of the exact sum (Higham), so of each other within 2x
        for k, ak in ((0, 1), (1, 1), (2, 3), (3, 3)):
            assert abs(got[k] - want[k]) <= 2 * n * EPS * want[ak] + 1e-300, (k, got, want)
    else:
        # Gaussians from the device libm: R(z) to m <= 23 bits absorbs nearly
        # every last-ulp difference; the rare flipped rounding moves a mean
        # by one residual / n
        np.testing.assert_allclose(got[[1, 3]], want[[1, 3]], rtol=1e-3)
        assert abs(got[0] - want[0]) <= 1e-3 * want[1]
        assert abs(got[2] - want[2]) <= 1e-3 * want[3]


def test_step_error_probe_errors_and_report(gpu):
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_step_error_report
    with pytest.raises(gpu.InvalidArgument):
        gpu.step_error_probe(gpu.make_gbm(), 3, gpu.PrecisionSpec.fp16_ieee(), None, 100, 1)
    bad = gpu.make_gbm(1e30, 0.0, 1e300)
    with pytest.raises(gpu.DomainError, match="non-finite operand") as ei:
        gpu.step_error_probe(bad, 2, gpu.PrecisionSpec.carrier(), None, 100, 1)
    assert ei.value.path_index == 0 and ei.value.step == 0
    cfg = ExperimentConfig(precisions=["fp16"], approx="linear:16", level_min=0, level_max=4)
    with pytest.raises(gpu.InvalidArgument, match="1e4 samples"):
        run_step_error_report(cfg, 9999)
    rows = run_step_error_report(cfg, 20000)
    assert [r.level for r in rows] == list(range(5))
    assert all(r.stats.samples == 20000 and r.stats.mean_abs_eta > 0 for r in rows)


# ------------------------------------------ density report (row 4, histogram) --
@pytest.mark.parametrize("idx", range(4))
def test_density_report_vs_reference(gpu, cv, idx):
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_density_report
    c = cv["density"][idx]
    width = float.fromhex(c["bin_width"])
    cfg = ExperimentConfig(approx=c["approx"], seed=c["seed"], level_min=0, level_max=0)
    rows = run_density_report(cfg, c["curve_points"], c["hist_samples"], width)
    want = c["rows"]
    assert len(rows) == len(want)
    got_kind = [0 if r.series == "curve" else 1 for r in rows]
    assert got_kind == [w[0] for w in want]
    gx = np.array([r.x for r in rows])
    gy = np.array([r.y for r in rows])
    wx = unhex([w[1] for w in want])
    wy = unhex([w[2] for w in want])
    kind = np.array(got_kind)
    assert np.array_equal(bits(gx[kind == 0]), bits(wx[kind == 0]))  # u grid: same arithmetic
    if c["approx"] != "exact":  # bin centres from the table's max_value: bitwise
        assert np.array_equal(bits(gx), bits(wx))
    else:  # centres from z_max = exact Z(1 - 2^-30): last-ulp
        np.testing.assert_allclose(gx, wx, rtol=1e-14, atol=1e-14)
    if c["approx"] != "exact":  # table values and integer counts: bitwise
        assert np.array_equal(bits(gy), bits(wy))
    else:  # device exact Gaussians: last-ulp curve; a draw may cross a bin edge
        cu = kind == 0
        np.testing.assert_allclose(gy[cu], wy[cu], rtol=1e-13, atol=1e-15)
        step = 1.0 / (c["hist_samples"] * width)
        assert np.max(np.abs(gy[~cu] - wy[~cu])) <= 3 * step + 1e-18
        assert abs(gy[~cu].sum() - wy[~cu].sum()) <= 1e-9


def test_multi_run_and_probe_range_fallback(gpu, ref):
    """Runs whose native fp32 legs leave the exact exponent range are re-run
    in the exact emulation inside a multi-run call and in the probe too."""
    P = gpu.PrecisionSpec
    hot = gpu.make_gbm(80.0, 0.2)  # EM growth (1 + 80/16)^16 > 2^33 at level 4
    tb = gpu.InvCdfApprox.parse("linear:16")
    runs = [(4, P.fp32(), True, 300, 0), (3, P.fp32(), False, 500, 7)]
    many = gpu.run_coupled_many(hot, tb, 2, runs)
    for (level, spec, kahan, n, base), m in zip(runs, many):
        one = gpu.run_coupled_paths(hot, level, spec, tb, kahan, n, 2, base)
        assert [m.d_hat.state(), m.d_bar.state(), m.d_four.state()] == \
               [one.d_hat.state(), one.d_bar.state(), one.d_four.state()]
    n = 20000
    got = gpu.step_error_probe(hot, 4, P.fp32(), tb, n, 5)
    rc, msg, want = ref.step_error_probe(level=4, mantissa_bits=23, approx="linear:16",
                                         n_samples=n, seed=5, mu=80.0)
    assert rc == 0, msg
    eps = 2.0 ** -52
    g = [got.mean_eta, got.mean_abs_eta, got.mean_eta_prime, got.mean_abs_eta_prime]
    for k, ak in ((0, 1), (1, 1), (2, 3), (3, 3)):
        assert abs(g[k] - want[k]) <= 2 * n * eps * want[ak] + 1e-300
