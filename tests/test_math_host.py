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
