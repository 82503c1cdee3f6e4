"""LPMC_EXACT_Z_GLIBC on the B200: the exact Gaussians restate glibc 2.39's
erfc/exp/log and the reference's own operation order (lpmc_glibc.cuh), so
everything the reference computes is reproduced bit for bit -- exact Z, all
four legs of every path, reference-order moments, LevelStats, the density
histogram of the exact transform, the step-error probe's residuals.  Golden
vectors come from the unmodified reference (tests/golden/); every call goes
through the C-ABI into liblpmc_b200.so.
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from conftest import ROOT, bits, unhex

pytestmark = pytest.mark.gpu

EPS = 2.0 ** -52
G = {"exact_z": "glibc"}


def _table(lib, name):
    return None if name == "exact" else lib.InvCdfApprox.parse(name)


@pytest.fixture(scope="module")
def cv():
    with open(os.path.join(ROOT, "tests", "golden", "callers_vectors.json")) as f:
        return json.load(f)


def test_glibc_z_golden_and_host(gpu, golden):
    """Device Z == the reference's Z (golden, both tails) == the host
    restatement, bitwise; the sampler grid's deepest tails included."""
    u = unhex(golden["gauss"]["u"])
    z = unhex(golden["gauss"]["z"])
    ok = (u > 0) & (u < 1)
    dev = gpu.device_inv_cdf(u[ok], exact_z="glibc")
    assert np.array_equal(bits(dev), bits(z[ok]))
    rng = np.random.default_rng(3)
    b = rng.integers(0, 1 << 53, 50000, dtype=np.uint64)
    k = 2 * np.arange(1, 2000, dtype=np.float64) + 1
    uu = np.concatenate([b.astype(np.float64) * 2.0 ** -53 + 2.0 ** -54, 2.0 ** -54 * k,
                         1.0 - 2.0 ** -54 * k])
    dev = gpu.api.device_math("exact_glibc", uu)
    host = np.array([gpu.api.glibc_math("inv_cdf", x) for x in uu])
    assert np.array_equal(bits(dev), bits(host))


@pytest.mark.parametrize("idx", range(0, 165))
def test_glibc_paths_bitexact(gpu, golden, idx):
    """All four legs of every golden path configuration (levels 0..7,
    m in {52,23,10,7,16,3,26}, exact and table Gaussians, +-Kahan) equal the
    reference's bitwise -- the hat legs included."""
    cases = golden["paths"]
    if idx >= len(cases):
        pytest.skip("fewer golden cases")
    c = cases[idx]
    want = unhex(c["out"]).reshape(-1, 4)
    out = gpu.simulate_paths(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                             _table(gpu, c["approx"]), bool(c["kahan"]), want.shape[0],
                             c["seed"], c["path_base"], **G)
    assert np.array_equal(bits(out), bits(want))


@pytest.mark.parametrize("idx", range(8))
def test_glibc_moments_bitexact(gpu, golden, idx):
    """Reference-order moments (d_hat, d_bar, d_four) of the golden runs,
    incl. the 2^20-path C1 checkpoint, bitwise."""
    c = golden["moments"][idx]
    want = [(a[0], *unhex(a[1:])) for a in c["acc"]]
    got = gpu.run_coupled_paths(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                                _table(gpu, c["approx"]), bool(c["kahan"]), c["n"], c["seed"],
                                c["path_base"], reduce="sequential", **G)
    assert [got.d_hat.state(), got.d_bar.state(), got.d_four.state()] == \
           [tuple(w) for w in want]


def test_glibc_level_stats_bitexact(gpu, golden):
    """estimate_level_stats (mlmc.hpp:113-149): every LevelStats field."""
    for c in golden["level_stats"]:
        want = unhex(c["out"])
        cost = gpu.CostModel(per_step_arithmetic=c["per_step_arithmetic"])
        s = gpu.estimate_level_stats(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                                     _table(gpu, c["approx"]), bool(c["kahan"]), c["n"], 1, cost,
                                     reduce="sequential", **G)
        got = [s.mean_hat, s.v_hat, s.v_hat_stderr, s.mean_bar, s.v_bar, s.v_bar_stderr,
               s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat, s.c_bar, s.C_bar, s.m_hat, s.m_bar,
               s.M_bar, s.level]
        assert np.array_equal(bits(got), bits(want))


def test_glibc_tree_moments_match_reference_paths(gpu, oracle, ref):
    """Tree mode on the reference's own per-path values: the GPU tree equals
    the restated tree of the paths the reference computes (ragged, two
    chunks, fp32 exact-Gaussian bar legs)."""
    level, n, base = 3, 262144 + 1001, 5
    rc, msg, paths = ref.simulate(level=level, mantissa_bits=23, approx="exact", kahan=True,
                                  seed=2, path_base=base, n=n)
    assert rc == 0, msg
    dh, db = paths[:, 0] - paths[:, 1], paths[:, 2] - paths[:, 3]
    got = gpu.run_coupled_paths(gpu.make_gbm(), level, gpu.PrecisionSpec.fp32(), None, True, n,
                                2, base, **G)
    assert [got.d_hat.state(), got.d_bar.state(), got.d_four.state()] == \
           oracle.tree_from_values(dh, db)


@pytest.mark.parametrize("idx", range(4))
def test_glibc_density_report_bitexact(gpu, cv, idx):
    """run_density_report (experiments.hpp:252-295) incl. the exact
    transform: curve and histogram rows bitwise."""
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_density_report
    c = cv["density"][idx]
    cfg = ExperimentConfig(approx=c["approx"], seed=c["seed"], level_min=0, level_max=0)
    rows = run_density_report(cfg, c["curve_points"], c["hist_samples"],
                              float.fromhex(c["bin_width"]), **G)
    got = np.array([[r.x, r.y] for r in rows])
    want = np.array([[float.fromhex(w[1]), float.fromhex(w[2])] for w in c["rows"]])
    assert np.array_equal(bits(got), bits(want))


@pytest.mark.parametrize("idx", range(8))
def test_glibc_step_error_probe(gpu, cv, idx):
    """step_error_probe (sde.hpp:297-344): identical residuals in every
    configuration, so the means agree to the summation-order bound."""
    c = cv["step_error"][idx]
    want = unhex(c["out"])
    n = c["n_samples"]
    r = gpu.step_error_probe(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                             _table(gpu, c["approx"]), n, c["seed"], **G)
    if n == 0:
        assert r.samples == 0
        return
    got = [r.mean_eta, r.mean_abs_eta, r.mean_eta_prime, r.mean_abs_eta_prime]
    for k, ak in ((0, 1), (1, 1), (2, 3), (3, 3)):
        assert abs(got[k] - want[k]) <= 2 * n * EPS * want[ak] + 1e-300, (k, got, want)


@pytest.mark.parametrize("idx", range(72))
def test_glibc_two_way_paths_bitexact(gpu, cv, idx):
    """simulate_two_way (sde.hpp:162-196): x_hat and x_bar bitwise."""
    c = cv["two_way_paths"][idx]
    want = unhex(c["out"]).reshape(-1, 2)
    out = gpu.simulate_paths(gpu.make_gbm(), c["level"], gpu.PrecisionSpec(c["m"]),
                             _table(gpu, c["approx"]), bool(c["kahan"]), want.shape[0], c["seed"],
                             c["path_base"], legs="fine", **G)
    assert np.array_equal(bits(out[:, [0, 2]]), bits(want))


def test_glibc_two_way_experiment_bitexact(gpu, cv):
    """run_two_way_experiment (experiments.hpp:79-147): every row bitwise."""
    from paper_2012_09739_b200.experiments import ExperimentConfig, run_two_way_experiment
    for row in cv["two_way_rows"]:
        cfg = ExperimentConfig(precisions=[row["precision"]], approx=row["approx"],
                               kahan=bool(row["kahan"]), level_min=row["level_min"],
                               level_max=row["level_max"], paths=[row["paths"]])
        got = run_two_way_experiment(cfg, reduce="sequential", **G)
        want = [unhex(r) for r in row["rows"]]
        assert len(got) == len(want)
        for g, w in zip(got, want):
            assert np.array_equal(bits([g.n_steps, g.variance, g.stderr_variance, g.paths]),
                                  bits(w))


@pytest.mark.parametrize("idx", range(4))
def test_glibc_nested_estimator_bitexact(gpu, cv, idx):
    """run_nested_estimator (mlmc.hpp:240-285): allocation, pilot statistics,
    level contributions, the estimate and the predicted times, bitwise."""
    n = cv["nested"][idx]
    r = gpu.run_nested_estimator(gpu.make_gbm(), n["max_level"], gpu.PrecisionSpec(n["m"]),
                                 _table(gpu, n["approx"]), bool(n["kahan"]),
                                 float.fromhex(n["eps"]), n["seed"],
                                 pilot_paths=n["pilot_paths"], reduce="sequential", **G)
    assert r.allocation.primary == n["primary"]
    assert r.allocation.secondary == n["secondary"]
    assert r.allocation.degenerate == n["degenerate"]
    pilot = unhex(n["pilot"]).reshape(-1, 16)
    for s, w in zip(r.pilot_stats, pilot):
        got = [s.mean_hat, s.v_hat, s.v_hat_stderr, s.mean_bar, s.v_bar, s.v_bar_stderr,
               s.mean_four, s.V_bar, s.V_bar_stderr, s.c_hat, s.c_bar, s.C_bar, s.m_hat,
               s.m_bar, s.M_bar, s.level]
        assert np.array_equal(bits(got), bits(w))
    assert np.array_equal(bits(r.level_contributions), bits(unhex(n["contributions"])))
    assert r.value == float.fromhex(n["value"])
    assert [r.times.t_hat, r.times.t_bar] == [float.fromhex(n["t_hat"]), float.fromhex(n["t_bar"])]
