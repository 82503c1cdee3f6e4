"""The reference's m = 7 (bf16) legs on native bfloat16 arithmetic
(dev::ArithBf16, lpmc_device.cuh): bfloat16 has fp32's exponent range, so the
native range guard of the fp32 policies is the whole exactness condition.

* the host's choice (lpmc_bar_arithmetic), CPU;
* on the B200: the production moments equal, bitwise, the restated reduction
  of the per-path values of the dump kernel (fp32-carried emulation, pinned
  to the reference by test_gpu_parity.py) -- every level parity, legs mask,
  table kind, +-Kahan, a model that leaves the native range (the launch is
  re-run in the binary64 emulation), and LPMC_NO_NATIVE_BF16 as the control.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import bits


def bf16(lib):
    return lib.PrecisionSpec(7, False)


def test_host_selects_native_bfloat16(lib):
    tb = lib.InvCdfApprox.parse("linear:16")
    for level in (0, 5, 12, 14):
        for kahan in (False, True):
            a = lib.api.bar_arithmetic(lib.make_gbm(), level, bf16(lib), tb, kahan)
            assert a["arith"] == "fp32-round" and a["native_bfloat16"], (level, a)
            assert not a["native_binary16"]
    a = lib.api.bar_arithmetic(lib.make_gbm(), 6, bf16(lib), lib.InvCdfApprox.parse("cubic:64"), True)
    assert a["native_bfloat16"]  # any table kind
    assert not lib.api.bar_arithmetic(lib.make_gbm(), 6, bf16(lib), tb, False,
                                      exact_z="glibc")["native_bfloat16"]
    assert not lib.api.bar_arithmetic(lib.make_gbm(), 6, lib.PrecisionSpec(10, False), tb,
                                      False)["native_bfloat16"]
    # constants outside the native range: the binary64 emulation
    a = lib.api.bar_arithmetic(lib.make_gbm(0.05, 1e-9, 1.0, 1.0), 6, bf16(lib), tb, False)
    assert a["arith"] == "fp64-round" and not a["native_bfloat16"]


def _check(gpu, oracle, model, level, approx, kahan, legs, payoff, n, seed, mu=0.05, sigma=0.2,
           x0=1.0, own_bar=True):
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    ext = {"legs": legs, "payoff": payoff, "strike": 1.0}
    out = gpu.simulate_paths(model, level, bf16(gpu), tb, kahan, n, seed, level << 40, **ext)
    if tb is not None and own_bar:  # the dump kernel's bar legs are the reference's own
        cfg = oracle.config(level=level, mantissa_bits=7, approx=approx, kahan=kahan, seed=seed,
                            mu=mu, sigma=sigma, x0=x0)
        own, _, fails = oracle.simulate(cfg, level << 40, n)
        assert not fails
        cols = slice(2, 3) if legs == "fine" else slice(2, 4)
        assert np.array_equal(bits(out[:, cols]), bits(own[:, cols]))
    pay = (lambda x: np.maximum(x - 1.0, 0.0)) if payoff == "call" else (lambda x: x)
    coarse = level > 0 and legs != "fine"
    dh = pay(out[:, 0]) - (pay(out[:, 1]) if coarse else 0.0)
    db = pay(out[:, 2]) - (pay(out[:, 3]) if coarse else 0.0)
    if legs == "bar":
        dh = np.zeros_like(db)
    want = oracle.tree_from_values(dh, db, legs={"all": 3, "bar": 2, "fine": 3}[legs])

    def moments():
        m = gpu.run_coupled_paths(model, level, bf16(gpu), tb, kahan, n, seed, level << 40, **ext)
        return [m.d_hat.state(), m.d_bar.state(), m.d_four.state()]

    assert moments() == want
    os.environ["LPMC_NO_NATIVE_BF16"] = "1"  # control: the fp32-carried emulation
    try:
        assert moments() == want
    finally:
        del os.environ["LPMC_NO_NATIVE_BF16"]


@pytest.mark.gpu
@pytest.mark.parametrize("kahan", [False, True])
@pytest.mark.parametrize("level", [0, 1, 2, 5, 6, 11, 12])
@pytest.mark.parametrize("approx", ["linear:16", "cubic:64", "exact"])
@pytest.mark.parametrize("legs,payoff", [("all", "call"), ("bar", "terminal"),
                                         ("fine", "terminal")])
def test_native_bfloat16_moments_bitexact(gpu, oracle, level, approx, legs, payoff, kahan):
    n = 3000 if level < 11 else 700
    _check(gpu, oracle, gpu.make_gbm(), level, approx, kahan, legs, payoff, n, 13)


@pytest.mark.gpu
@pytest.mark.parametrize("kahan", [False, True])
@pytest.mark.parametrize("level", [2, 6])
@pytest.mark.parametrize("mu,sigma,x0", [(0.05, 3.0, 1.0),    # sign changes, wide magnitudes
                                         (80.0, 0.2, 1.0),    # leaves [2^-32, 2^33): re-run exactly
                                         (-0.75, 0.5, 300.0)])
def test_native_bfloat16_wide_models(gpu, oracle, level, mu, sigma, x0, kahan):
    model = gpu.make_gbm(mu, sigma, x0, 1.0)
    _check(gpu, oracle, model, level, "linear:16", kahan, "all", "terminal", 3000, 4, mu=mu,
           sigma=sigma, x0=x0)


@pytest.mark.gpu
def test_native_bfloat16_full_chunk(gpu, oracle):
    _check(gpu, oracle, gpu.make_gbm(), 8, "linear:16", True, "all", "call", 262144 + 300, 1,
           own_bar=False)
