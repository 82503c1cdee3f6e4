"""Accuracy of the device erfc core (lpmc_math.cuh), evaluated on the host
(lpmc_erfc_core is the same IEEE fma/mul/add sequence, so bitwise the device
result; tests/test_gpu_parity.py checks that identity on a B200), against
mpmath at 40 digits, with glibc's erfc (what the reference calls,
gaussian.hpp:15) measured the same way for comparison.  CPU only."""
from __future__ import annotations

import ctypes
import ctypes.util
import math

import mpmath as mp
import numpy as np
import pytest

mp.mp.dps = 40
_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.erfc.restype = ctypes.c_double
_libm.erfc.argtypes = [ctypes.c_double]


def ulp_err(got: float, t: float) -> float:
    exact = mp.erfc(mp.mpf(t))
    return float(abs(mp.mpf(got) - exact) / mp.mpf(math.ulp(float(exact))))


@pytest.fixture(scope="module")
def samples():
    rng = np.random.default_rng(2024)
    t = np.concatenate([rng.uniform(0.0, 6.5, 3000), rng.uniform(0.0, 1.0, 1000),
                        np.arange(0, 26) * 0.25, np.arange(0, 26) * 0.25 + 0.125,
                        np.nextafter(np.arange(1, 26) * 0.25, 0)])
    # the sampler's actual arguments: t = (-x) / sqrt(2) for x ~ N(0, 1), x <= 0
    x = -np.abs(rng.standard_normal(3000))
    t2 = -x * 0.7071067811865475244
    return np.concatenate([t, t2[t2 < 6.5]])


def test_erfc_core_accuracy(lib, samples):
    errs = np.array([ulp_err(lib.api.erfc_core(t), t) for t in samples])
    glibc = np.array([ulp_err(_libm.erfc(t), t) for t in samples])
    print(f"\nerfc core: max {errs.max():.3f} ulp, mean {errs.mean():.3f}, "
          f"correctly rounded {np.mean(errs <= 0.5):.3f}; glibc: max {glibc.max():.3f}, "
          f"mean {glibc.mean():.3f}, correctly rounded {np.mean(glibc <= 0.5):.3f}")
    assert errs.max() <= 2.0
    assert errs.mean() <= 0.6


def test_erfc_core_domain_edges(lib):
    assert lib.api.erfc_core(0.0) == 1.0
    # outside the fast range the host hook falls back to libm; never NaN
    for t in (6.5, 10.0, 27.0):
        assert math.isfinite(lib.api.erfc_core(t))


# ---- the direct table of the default exact inverse CDF ----------------------
def _ndtri_lower(v):
    return -mp.sqrt(2) * mp.erfinv(1 - 2 * mp.mpf(v))


def _unit(v, z):
    """eps (v / pdf(z) + |z|): the conditioning of Z on a 1-ulp error of u
    plus one ulp of Z (the unit of tests/test_gpu_parity.py's Z bound)."""
    pdf = mp.exp(-z * z / 2) / mp.sqrt(2 * mp.pi)
    return mp.mpf(2) ** -52 * (mp.mpf(v) / pdf + abs(z))


def test_direct_table_accuracy(lib):
    """Phi^-1 from the direct table (bitwise the device's evaluation) against
    mpmath: at most 0.6 units (measured 0.41: the final addition's half ulp),
    on the sampler's grid, at every sub-interval edge and one grid step either
    side of it."""
    rng = np.random.default_rng(11)
    b = rng.integers(0, 1 << 52, 4000, dtype=np.uint64)  # u < 1/2: v = u
    v = [(float(x) + 0.5) * 2.0 ** -53 for x in b]
    for e in range(1, 15):  # binades [2^-(e+1), 2^-e): 32 sub-intervals each
        lo = 2.0 ** -(e + 1)
        for sub in range(32):
            a = lo * (1 + sub / 32)
            v += [a, np.nextafter(a, 1.0), np.nextafter(a, 0.0)]
    worst = 0.0
    n = 0
    for x in v:
        z = lib.api.phi_inv_direct_core(float(x))
        if z is None:
            assert x < 2.0 ** -15
            continue
        zt = _ndtri_lower(x)
        worst = max(worst, float(abs(mp.mpf(z) - zt) / _unit(x, zt)))
        n += 1
    print(f"\ndirect table: max normalised error {worst:.3f} over {n} points")
    assert n > 5000 and worst <= 0.6


def test_direct_table_edges(lib):
    z = lib.api.phi_inv_direct_core(0.5)
    assert z == 0.0 and math.copysign(1.0, z) == 1.0  # gaussian.hpp:62: exactly +0
    assert lib.api.phi_inv_direct_core(2.0 ** -15) is not None
    assert lib.api.phi_inv_direct_core(np.nextafter(2.0 ** -15, 0.0)) is None
    for bad in (0.0, -1.0, 0.75, float("nan")):
        assert lib.api.phi_inv_direct_core(bad) is None
    # monotone across sub-interval and binade edges
    for e in range(1, 15):
        for sub in range(32):
            a = 2.0 ** -(e + 1) * (1 + sub / 32)
            below = np.nextafter(a, 0.0)
            if below < 2.0 ** -15:
                continue
            assert lib.api.phi_inv_direct_core(below) <= lib.api.phi_inv_direct_core(a)


# ---- index arithmetic of the level kernel's dyadic-table lookup -------------
def test_reversed_dyadic_index_matches_reference_index():
    """approx_inv_up (lpmc_device.cuh) reads record r = e' - 969 of a reversed
    table copy, e' the biased exponent of (1 - 2^-53) - u', with an unsigned
    minimum at 53; record r <= 52 holds interval j = 52 - r.  For every
    reflected draw u' in [1/2, 1] on the 2^-53 grid this must be the
    reference's j = floor(-log2(1 - u')) - 1 (invcdf_approx.hpp:52-66), with
    v = 0 and v = 2^-53 landing on tail records.  Checked at every binade
    edge +-48 grid steps and on random grid points (numpy bit arithmetic, the
    same operations as the device's)."""
    g = 2.0 ** -53
    pts = [0.5, 1.0, 1.0 - g, 1.0 - 2 * g]
    for k in range(1, 53):
        edge = 1.0 - 2.0 ** -k  # u' where v = 2^-k exactly
        pts += [edge + i * g for i in range(-48, 49) if 0.5 <= edge + i * g <= 1.0]
    rng = np.random.default_rng(17)
    pts += list(0.5 + rng.integers(0, 1 << 52, 20000).astype(np.float64) * g)
    up = np.array(pts, dtype=np.float64)
    vm = np.float64(1.0 - g) - up  # exact: both on the 2^-53 grid
    hi = (vm.view(np.uint64) >> np.uint64(32)).astype(np.uint64)
    r = np.minimum(((hi >> np.uint64(20)) - np.uint64(969)) & np.uint64(0xFFFFFFFF), np.uint64(53))
    v = 1.0 - up  # exact
    for ri, vi in zip(r.tolist(), v.tolist()):
        if vi == 0.0:
            assert ri == 53  # u' == 1: a tail record (the sign bit of vm wraps the index)
            continue
        m, e = math.frexp(vi)  # vi = m 2^e, m in [1/2, 1)
        fl = -e + 1 if m == 0.5 else -e  # floor(-log2 v)
        j = fl - 1
        assert 0 <= j <= 52
        if vi == g:  # vm == 0: exponent field 0 wraps onto record 53, a copy of j = 52 (tail)
            assert j == 52 and ri == 53
            continue
        assert ri == 52 - j, (vi, ri, j)
