"""Bitwise agreement of the device exact Gaussians with glibc's (the
reference's libm) by |z| range, on the sampler's uniform grid.

    python tools/z_agreement.py [n]
"""
from __future__ import annotations

import ctypes
import ctypes.util
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2012_09739_b200 import api  # noqa: E402

libm = ctypes.CDLL(ctypes.util.find_library("m"))
libm.erfc.restype = ctypes.c_double
libm.erfc.argtypes = [ctypes.c_double]
libm.exp.restype = ctypes.c_double
libm.exp.argtypes = [ctypes.c_double]
libm.log.restype = ctypes.c_double
libm.log.argtypes = [ctypes.c_double]


def ref_inv_cdf(u: float) -> float:
    """gaussian.hpp:26-65 with glibc, scalar (the oracle's formula)."""
    if u == 0.5:
        return 0.0
    v = 1.0 - u if u > 0.5 else u
    a = [-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
         1.383577518672690e+02, -3.066479806614716e+01, 2.506628277459239e+00]
    b = [-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
         6.680131188771972e+01, -1.328068155288572e+01]
    c = [-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
         -2.549732539343734e+00, 4.374664141464968e+00, 2.938163982698783e+00]
    d = [7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
         3.754408661907416e+00]
    if v < 0.02425:
        q = (-2.0 * libm.log(v)) ** 0.5
        x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) / \
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1.0)
    else:
        q = v - 0.5
        r = q * q
        x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q / \
            (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1.0)
    err = 0.5 * libm.erfc(-x * 0.7071067811865475244) - v
    x -= err / (0.3989422804014326779 * libm.exp(-0.5 * x * x))
    return -x if u > 0.5 else x


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
    rng = np.random.default_rng(77)
    b = rng.integers(0, 1 << 53, n, dtype=np.uint64)
    u = b.astype(np.float64) * 2.0 ** -53 + 2.0 ** -54
    zr = np.array([ref_inv_cdf(x) for x in u])
    zd = api.device_math("exact", u)
    eq = zd.view(np.uint64) == zr.view(np.uint64)
    az = np.abs(zr)
    print(f"all: {eq.mean():.4f} of {n}")
    for lo, hi in [(0, 0.1), (0.1, 0.5), (0.5, 1), (1, 1.5), (1.5, 2), (2, 3), (3, 9)]:
        m = (az >= lo) & (az < hi)
        print(f"|z| in [{lo}, {hi}): {eq[m].mean():.4f} ({m.sum()} draws)")


if __name__ == "__main__":
    main()
