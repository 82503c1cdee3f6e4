"""The bar arithmetic for m <= 10 (ArithF32Round, lpmc_device.cuh) rounds an
fp32 result to m + 1 significant bits with Veltkamp's split in round-to-
nearest-even fp32 arithmetic, c = x (2^d + 1), hi = c - (c - x), d = 23 - m.
It must equal the integer RNE of the bit pattern (the reference's
round_to_precision on an fp32-representable value, softfloat.hpp:69-80) for
every m >= 1 the library accepts, ties included, over the normal range the
native range guard allows.  numpy float32 operations round like the device's
__fmul_rn / __fsub_rn."""
from __future__ import annotations

import numpy as np
import pytest


def rne_int(x: np.ndarray, d: int) -> np.ndarray:
    b = x.view(np.uint32).astype(np.uint64)
    b = (b + ((1 << (d - 1)) - 1) + ((b >> d) & 1)) & ~np.uint64((1 << d) - 1)
    return b.astype(np.uint32).view(np.float32)


def veltkamp(x: np.ndarray, d: int) -> np.ndarray:
    c = (x * np.float32((1 << d) + 1)).astype(np.float32)
    t = (c - x).astype(np.float32)
    return (c - t).astype(np.float32)


@pytest.mark.parametrize("m", list(range(1, 11)) + [16, 20])
def test_veltkamp_equals_integer_rne(m):
    d = 23 - m
    rng = np.random.default_rng(m)
    n = 400_000
    # exponents inside the native range guard's reach (2^-100 .. 2^60)
    e = rng.integers(127 - 100, 127 + 60, n, dtype=np.uint32)
    mant = rng.integers(0, 1 << 23, n, dtype=np.uint32)
    tie = rng.random(n) < 0.4  # exact ties: the dropped bits are 100...0
    mant = np.where(tie, (mant & ~np.uint32((1 << d) - 1)) | np.uint32(1 << (d - 1)), mant)
    edge = rng.random(n) < 0.1  # all-ones mantissas: rounding carries into the exponent
    mant = np.where(edge, np.uint32((1 << 23) - 1), mant)
    sign = (rng.random(n) < 0.5).astype(np.uint32) << 31
    x = (sign | (e << 23) | mant).view(np.float32)
    x = np.concatenate([x, np.float32([0.0, -0.0, 1.0, -1.0, 1.5, 2.5, 3.5])])
    with np.errstate(over="raise", under="raise"):
        got = veltkamp(x, d)
    assert np.array_equal(got.view(np.uint32), rne_int(x, d).view(np.uint32))


def rne_int64(x: np.ndarray, d: int) -> np.ndarray:
    b = x.view(np.uint64)
    b = (b + np.uint64((1 << (d - 1)) - 1) + ((b >> np.uint64(d)) & np.uint64(1))) & \
        ~np.uint64((1 << d) - 1)
    return b.view(np.float64)


@pytest.mark.parametrize("m", [1, 3, 7, 10])
def test_veltkamp_binary64_lift(m):
    """ArithF32Round::lift: R(z) of a binary64 Gaussian (0 or normal, |z| < 40)
    to m + 1 bits by Veltkamp's split in binary64 (d = 52 - m)."""
    d = 52 - m
    rng = np.random.default_rng(100 + m)
    n = 400_000
    z = rng.standard_normal(n) * np.exp2(rng.integers(-60, 3, n))
    b = z.view(np.uint64)
    tie = rng.random(n) < 0.4
    b = np.where(tie, (b & ~np.uint64((1 << d) - 1)) | np.uint64(1 << (d - 1)), b)
    z = np.concatenate([b.view(np.float64), [0.0, -0.0, 4.3153065737391225, -8.3]])
    c = z * float((1 << d) + 1)
    got = c - (c - z)
    assert np.array_equal(got.view(np.uint64), rne_int64(z, d).view(np.uint64))
