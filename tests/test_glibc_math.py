"""The glibc restatement behind LPMC_EXACT_Z_GLIBC (lpmc_glibc.cuh), on the
host (the same IEEE operation sequence as the device, checked bitwise on the
B200 by test_gpu_glibc.py):

* exp / log / erfc bitwise equal to the running glibc libm (the library the
  reference links, gaussian.hpp:15,19,45) over the sampler's argument ranges
  and beyond;
* exact_inv_cdf (gaussian.hpp:59-65) bitwise equal to the reference's, on
  the golden vectors and, where oracle/_ref is built, on the sampler's grid
  down to u = 2^-54.

CPU only.  The restatement is pinned to the libm of this image (sha256 in
lpmc_glibc_coef.h); on another libm the libm comparisons skip.
"""
from __future__ import annotations

import ctypes
import ctypes.util
import hashlib
import os
import re

import numpy as np
import pytest

from conftest import ROOT, bits, unhex

_libm = ctypes.CDLL(ctypes.util.find_library("m"))
for _f in ("exp", "log", "erfc"):
    getattr(_libm, _f).restype = ctypes.c_double
    getattr(_libm, _f).argtypes = [ctypes.c_double]


def _pinned_sha() -> str:
    with open(os.path.join(ROOT, "paper_2012_09739_b200", "csrc", "lpmc_glibc_coef.h")) as f:
        return re.search(r"sha256 ([0-9a-f]{64})", f.read()).group(1)


def _running_libm_sha() -> str | None:
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from glibc_constants import libm_path
    try:
        with open(libm_path(), "rb") as f:
            return hashlib.sha256(f.read()).hexdigest()
    except OSError:
        return None


@pytest.fixture(scope="module")
def same_libm():
    if _running_libm_sha() != _pinned_sha():
        pytest.skip("running libm is not the pinned glibc 2.39 build")


def _compare(lib, op: str, xs: np.ndarray):
    got, want, skipped = [], [], 0
    for x in xs:
        r = lib.api.glibc_math(op, float(x))
        if r is None:
            skipped += 1
            continue
        got.append(r)
        want.append(getattr(_libm, op)(float(x)))
    got, want = np.array(got), np.array(want)
    bad = np.nonzero(bits(got) != bits(want))[0]
    assert bad.size == 0, f"{op}: {bad.size} mismatches, first {got[bad[0]].hex()} vs " \
                          f"{want[bad[0]].hex()}"
    return len(got), skipped


def test_glibc_exp_bitwise(lib, same_libm):
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(-36.0, 0.0, 60000),          # pdf and erfc arguments
                         rng.uniform(-1.0, 1.0, 20000), rng.uniform(-1e-6, 1e-6, 5000),
                         rng.uniform(-700.0, 700.0, 5000), [0.0, -0.0, 2.0 ** -60]])
    n, skipped = _compare(lib, "exp", xs)
    assert skipped < 0.05 * len(xs) and n > 80000


def test_glibc_log_bitwise(lib, same_libm):
    rng = np.random.default_rng(12)
    xs = np.concatenate([2.0 ** rng.uniform(-54.0, -5.36, 60000),  # Acklam's tail, v < 0.02425
                         rng.uniform(0.0, 1.0, 10000), 2.0 ** rng.uniform(-1000, 1000, 10000)])
    n, skipped = _compare(lib, "log", xs)
    assert n > 70000


def test_glibc_erfc_bitwise(lib, same_libm):
    rng = np.random.default_rng(13)
    xs = np.concatenate([rng.uniform(0.0, 6.0, 60000),            # t = -x0 / sqrt 2
                         rng.uniform(-6.5, 6.5, 20000), rng.uniform(0.0, 0.3, 5000),
                         np.array([0.84375, 1.25, 1 / 0.35, 6.0, 2.0 ** -57, 0.25, -0.0]),
                         np.nextafter(np.array([0.84375, 1.25, 1 / 0.35, 0.25]), 0)])
    n, skipped = _compare(lib, "erfc", xs)
    assert skipped == 0 and n == len(xs)


def test_glibc_inv_cdf_golden(lib, golden):
    """exact_inv_cdf on the golden uniforms (both tails, u = 1/2): bitwise the
    reference's Z (tests/golden/reference_vectors.json, from oracle/_ref)."""
    u = unhex(golden["gauss"]["u"])
    z = unhex(golden["gauss"]["z"])
    ok = (u > 0) & (u < 1)
    got = np.array([lib.api.glibc_math("inv_cdf", x) for x in u[ok]])
    assert np.array_equal(bits(got), bits(z[ok]))


def test_glibc_inv_cdf_reference_grid(lib, ref):
    """On the sampler's grid u = b 2^-53 + 2^-54, random draws plus the
    deepest tails on both sides: bitwise the reference's exact_inv_cdf."""
    rng = np.random.default_rng(14)
    b = rng.integers(0, 1 << 53, 100000, dtype=np.uint64)
    u = b.astype(np.float64) * 2.0 ** -53 + 2.0 ** -54
    k = 2 * np.arange(1, 3000, dtype=np.float64) + 1
    u = np.concatenate([u, 2.0 ** -54 * k, 1.0 - 2.0 ** -54 * k, [0.02425, 0.5, 0.25]])
    want = ref.exact_inv_cdf(u)
    got = np.array([lib.api.glibc_math("inv_cdf", x) for x in u])
    assert np.array_equal(bits(got), bits(want))
