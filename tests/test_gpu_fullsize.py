"""BASELINE.json's configurations at their full sizes, checked through
properties that do not need the oracle to simulate the whole run:

* last-chunk parity: the run's final (ragged) 2^18-path chunk, at path
  indices up to 2^30 + 999 inside a level (C5), is computed by the device
  alone (lpmc_level_partials, include/lpmc_b200.h) and must equal the
  oracle's restated chunk tree bitwise -- with exact_z="glibc" for the
  configurations that carry exact legs (then every leg is the reference's);
* split invariance at 2^30 paths: partials of any two chunk ranges
  concatenate to the whole run's, and their index-order fold is the
  run_coupled_paths result (mlmc.hpp:108-110);
* fast vs glibc exact Gaussians at full size: the bar legs never see the
  exact Gaussian, so d_bar is bitwise equal in both modes; d_hat and d_four
  agree within the fast mode's stated tolerances (test_gpu_parity.py);
* level 0 at 2^30 paths: X_1 = x0 (1 + mu) + x0 sigma Z, so mean and
  variance of d_hat are known in closed form (6-sigma statistical bound).
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

CHUNK = 262144  # paths per chunk accumulator (lpmc_internal.h)
G = {"exact_z": "glibc"}


def _table(lib, name):
    return None if name == "exact" else lib.InvCdfApprox.parse(name)


# (name, level, mantissa_bits, ieee_half, approx, kahan, legs, payoff, n_paths, glibc)
LAST_CHUNK = [
    ("C1", 6, 52, False, "exact", False, "all", "terminal", (1 << 20) + 12345, True),
    ("C2", 10, 23, False, "linear:16", False, "all", "terminal", (1 << 22) + 777, True),
    ("C2+K", 10, 23, False, "linear:16", True, "all", "terminal", (1 << 22) + 777, True),
    ("C3-ieee", 8, 10, True, "constant:16", True, "bar", "terminal", (1 << 24) + 1001, False),
    ("C3-ieee", 8, 10, True, "linear:16", False, "bar", "terminal", (1 << 24) + 1001, False),
    ("C3-ref", 8, 10, False, "linear:16", True, "bar", "terminal", (1 << 24) + 1001, False),
    ("C4-fp16", 12, 10, False, "linear:16", False, "all", "call", (1 << 24) + 513, True),
    ("C4-fp32", 12, 23, False, "linear:16", True, "all", "call", (1 << 24) + 513, True),
    ("C5-fp64", 14, 52, False, "linear:16", True, "all", "terminal", (1 << 30) + 99, True),
    ("C5-fp16", 14, 10, False, "linear:16", True, "all", "call", (1 << 30) + 99, True),
    ("C5-ieee", 14, 10, True, "linear:16", True, "bar", "terminal", (1 << 30) + 99, False),
]
LEGS = {"hat": 1, "bar": 2, "all": 3}
PAYOFF = {"terminal": 0, "call": 1}


@pytest.mark.parametrize("case", LAST_CHUNK, ids=[f"{c[0]}-{c[4]}-K{int(c[5])}" for c in LAST_CHUNK])
def test_last_chunk_bitwise_at_full_size(gpu, oracle, case):
    """The final ragged chunk of a full-size run (path offsets up to 2^30
    inside the level, path_base = level << 40 as experiments.hpp:185) equals
    the oracle's chunk tree of the same paths bitwise."""
    name, level, m, ieee, approx, kahan, legs, payoff, n, glibc = case
    model = gpu.make_gbm()
    base = level << 40
    last = (n - 1) // CHUNK
    ext = {"legs": legs, "payoff": payoff, "strike": 1.0}
    if glibc:
        ext.update(G)
    got = gpu.level_partials(model, level, gpu.PrecisionSpec(m, ieee), _table(gpu, approx), kahan,
                             n, 1, base, last, last + 1, **ext)
    cfg = oracle.config(level=level, mantissa_bits=m, approx=approx, kahan=kahan, seed=1,
                        ieee_half=ieee, legs=LEGS[legs], payoff=PAYOFF[payoff], strike=1.0)
    want = oracle.chunk_partials(cfg, n, base, last, last + 1)
    assert got[0, 1 if legs == "bar" else 0, 0] == n - last * CHUNK  # d_hat unused by bar-only
    assert np.array_equal(bits(got), bits(want)), name


@pytest.mark.parametrize("cut", [1, 1234, 4095])
def test_two_to_thirty_paths_split_bitwise(gpu, cut):
    """C5 path count (2^30 per level): partials over [0, cut) and
    [cut, 4096) concatenate to the whole run's bitwise; the fold is
    run_coupled_paths' result; every accumulator counts 2^30 paths."""
    model = gpu.make_gbm()
    n = 1 << 30
    args = (model, 1, gpu.PrecisionSpec.fp16(), gpu.InvCdfApprox.parse("linear:16"), True, n, 1,
            1 << 40)
    nc = n // CHUNK
    whole = gpu.level_partials(*args, 0, nc)
    a = gpu.level_partials(*args, 0, cut)
    b = gpu.level_partials(*args, cut, nc)
    assert np.array_equal(bits(np.concatenate([a, b])), bits(whole))
    run = gpu.run_coupled_paths(*args)
    folded = gpu.fold_partials(whole)
    for f, r in ((folded.d_hat, run.d_hat), (folded.d_bar, run.d_bar),
                 (folded.d_four, run.d_four)):
        assert f.state() == r.state()
        assert r.count() == n


def test_level0_two_to_thirty_closed_form(gpu):
    """Level 0, 2^30 paths, fp64 exact: d_hat = X_1 = x0 (1 + mu) + x0 sigma Z
    (one EM step, coarse := 0, sde.hpp:247), so E = 1.05 and Var = 0.04."""
    model = gpu.make_gbm()
    n = 1 << 30
    m = gpu.run_coupled_paths(model, 0, gpu.PrecisionSpec.carrier(), None, False, n, 1, 0,
                              legs="hat")
    sd = 0.2
    assert abs(m.d_hat.mean() - 1.05) <= 6 * sd / math.sqrt(n)
    # Var of the sample variance of a Gaussian: 2 sigma^4 / (n - 1)
    assert abs(m.d_hat.variance() - sd * sd) <= 6 * math.sqrt(2.0 / (n - 1)) * sd * sd
    assert abs(m.d_hat.variance_stderr() - math.sqrt(2.0 / n) * sd * sd) <= 2e-3 * sd * sd


# (name, level, mantissa_bits, approx, kahan, payoff, n_paths)
FULL = [
    ("C1", 6, 52, "exact", False, "terminal", 1 << 20),
    ("C2", 10, 23, "linear:16", False, "terminal", 1 << 22),
    ("C2+K", 10, 23, "linear:16", True, "terminal", 1 << 22),
    ("C3-ref-lin+K", 8, 10, "linear:16", True, "terminal", 1 << 24),
    ("C3-ref-const", 8, 10, "constant:16", False, "terminal", 1 << 24),
    ("C4-fp16", 12, 10, "linear:16", False, "call", 1 << 24),
    ("C4-fp32", 12, 23, "linear:16", False, "call", 1 << 24),
    ("C4-fp32+K", 12, 23, "linear:16", True, "call", 1 << 24),
    ("C5-l14", 14, 23, "linear:16", True, "terminal", 1 << 22),
]


@pytest.mark.parametrize("case", FULL, ids=[c[0] for c in FULL])
def test_fast_vs_glibc_full_size(gpu, case):
    """The two exact-Gaussian modes at full size: glibc mode is bitwise the
    reference (test_gpu_glibc.py), so this checks the fast (default, bench)
    mode against the reference's own numbers at the sizes BASELINE names."""
    name, level, m, approx, kahan, payoff, n = case
    model = gpu.make_gbm()
    sp, tb = gpu.PrecisionSpec(m, False), _table(gpu, approx)
    base = level << 40
    fast = gpu.run_coupled_paths(model, level, sp, tb, kahan, n, 1, base, payoff=payoff)
    ref = gpu.run_coupled_paths(model, level, sp, tb, kahan, n, 1, base, payoff=payoff, **G)
    for f, r in ((fast.d_hat, ref.d_hat), (fast.d_four, ref.d_four)):
        assert f.count() == r.count() == n
    vh = ref.d_hat.variance()
    assert abs(fast.d_hat.variance() - vh) <= 1e-12 * vh, name
    assert abs(fast.d_hat.mean() - ref.d_hat.mean()) <= 1e-12 * math.sqrt(vh), name
    if tb is None:
        # exact bar legs: with m = 52 the bar legs are the hat legs, d_four == 0
        assert fast.d_four.variance() == ref.d_four.variance() == 0.0
        assert fast.d_four.mean() == ref.d_four.mean() == 0.0
    else:
        assert fast.d_bar.state() == ref.d_bar.state(), name  # no exact Z in the bar legs
        v4 = ref.d_four.variance()
        assert abs(fast.d_four.variance() - v4) <= 1e-10 * v4, name
        assert abs(fast.d_four.mean() - ref.d_four.mean()) <= 1e-12 * math.sqrt(v4), name
