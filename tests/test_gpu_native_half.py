"""The reference's m = 10 emulation on native binary16 arithmetic with static
power-of-two scales (dev::ArithHalfScaled, lpmc_device.cuh): production
launches with or without Kahan compensation, fast exact Gaussians,
dyadic-linear tables or none.

* the host's choice (lpmc_bar_arithmetic) for the BASELINE configurations and
  for models outside the proof's conditions (CPU);
* on the B200: the production moments equal, bitwise, the restated reduction
  of the per-path values of the dump kernel (fp32-carried emulation, pinned to
  the reference by test_gpu_parity.py) -- at every level parity, for every
  legs mask, with models that push paths out of the native guard (those paths
  are replayed in the emulation inside the kernel), and with the native path
  disabled as a control (LPMC_NO_NATIVE_HALF).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import bits


def fp16(lib):
    return lib.PrecisionSpec(10, False)


def test_host_selects_native_binary16_for_baseline_levels(lib):
    tb = lib.InvCdfApprox.parse("linear:16")
    for level in range(0, 15):  # BASELINE configs 3-5: T = 1, levels 0..14
        a = lib.api.bar_arithmetic(lib.make_gbm(), level, fp16(lib), tb, False)
        assert a["arith"] == "fp32-round" and a["native_binary16"], (level, a)
        assert a["pow2_folded"] == (level % 2 == 0), (level, a)
    # exact Gaussians for the low-precision legs (no table) qualify as well
    assert lib.api.bar_arithmetic(lib.make_gbm(), 6, fp16(lib), None, False)["native_binary16"]


def test_host_falls_back_outside_the_proof(lib):
    tb = lib.InvCdfApprox.parse("linear:16")
    nat = lambda **kw: lib.api.bar_arithmetic(kw.pop("model", lib.make_gbm()), kw.pop("level", 6),
                                              kw.pop("spec", fp16(lib)), kw.pop("tb", tb),
                                              kw.pop("kahan", False), **kw)["native_binary16"]
    assert nat()
    assert nat(kahan=True)                                       # with or without Kahan
    assert not nat(model=lib.make_gbm(0.05, 0.2, 1.0, 0.75))     # dt not a power of two
    assert not nat(model=lib.make_gbm(0.0, 0.2, 1.0, 1.0))       # mu == 0: no mantissa
    assert not nat(model=lib.make_gbm(0.05, 0.2, 1e-3, 1.0))     # x0 below the guard
    assert not nat(model=lib.make_gbm(0.05, 1e-5, 1.0, 1.0))     # scales out of binary16's range
    assert not nat(spec=lib.PrecisionSpec(7, False))             # bf16-like: m != 10
    assert not nat(spec=lib.PrecisionSpec.fp32())
    assert not nat(tb=lib.InvCdfApprox.parse("cubic:16"))        # not a dyadic-linear table
    assert not nat(exact_z="glibc")
    assert not nat(legs="hat")


def _moments(gpu, model, level, tb, n, seed, base, kahan=False, **ext):
    m = gpu.run_coupled_paths(model, level, fp16(gpu), tb, kahan, n, seed, base, **ext)
    return [m.d_hat.state(), m.d_bar.state(), m.d_four.state()]


def _want(gpu, oracle, model, level, tb, n, seed, base, legs="all", payoff="terminal",
          kahan=False):
    ext = {"legs": legs, "payoff": payoff, "strike": 1.0}
    out = gpu.simulate_paths(model, level, fp16(gpu), tb, kahan, n, seed, base, **ext)
    pay = (lambda x: np.maximum(x - 1.0, 0.0)) if payoff == "call" else (lambda x: x)
    coarse = level > 0 and legs != "fine"
    dh = pay(out[:, 0]) - (pay(out[:, 1]) if coarse else 0.0)
    db = pay(out[:, 2]) - (pay(out[:, 3]) if coarse else 0.0)
    if legs == "bar":
        dh = np.zeros_like(db)
    return out, oracle.tree_from_values(dh, db, legs={"all": 3, "bar": 2, "fine": 3}[legs])


@pytest.mark.gpu
@pytest.mark.parametrize("kahan", [False, True])
@pytest.mark.parametrize("level", [0, 1, 2, 3, 6, 7, 11, 12])
@pytest.mark.parametrize("approx", ["linear:16", "linear:4", "exact"])
@pytest.mark.parametrize("legs,payoff", [("all", "call"), ("bar", "terminal"),
                                         ("fine", "terminal")])
def test_native_binary16_moments_bitexact(gpu, oracle, level, approx, legs, payoff, kahan):
    n = 3000 if level < 11 else 700
    model = gpu.make_gbm()
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    assert gpu.api.bar_arithmetic(model, level, fp16(gpu), tb, kahan, legs=legs)["native_binary16"]
    out, want = _want(gpu, oracle, model, level, tb, n, 11, level << 40, legs, payoff, kahan)
    if tb is not None:  # the dump kernel's bar legs are the reference's own
        cfg = oracle.config(level=level, mantissa_bits=10, approx=approx, kahan=kahan, seed=11)
        own, _, _ = oracle.simulate(cfg, level << 40, n)
        cols = slice(2, 3) if legs == "fine" else slice(2, 4)
        assert np.array_equal(bits(out[:, cols]), bits(own[:, cols]))
    ext = {"legs": legs, "payoff": payoff, "strike": 1.0}
    assert _moments(gpu, model, level, tb, n, 11, level << 40, kahan, **ext) == want
    os.environ["LPMC_NO_NATIVE_HALF"] = "1"  # control: the fp32-carried emulation
    try:
        assert _moments(gpu, model, level, tb, n, 11, level << 40, kahan, **ext) == want
    finally:
        del os.environ["LPMC_NO_NATIVE_HALF"]


@pytest.mark.gpu
@pytest.mark.parametrize("kahan", [False, True])
@pytest.mark.parametrize("level", [2, 5, 8])
@pytest.mark.parametrize("mu,sigma,x0", [(0.05, 3.0, 1.0),      # sign changes, |x| down to 0
                                         (0.05, 0.2, 0.0703125),  # x0 just above the guard's 2^-4
                                         (0.05, 0.9, 4000.0),   # scaled products overflow binary16
                                         (-0.75, 0.5, 1.0),     # negative drift mantissa
                                         (0.05, 0.2, 1.0)])
def test_native_binary16_guard_replays_are_exact(gpu, oracle, level, mu, sigma, x0, kahan):
    """Models whose paths leave the native guard (|x| outside [2^-4, 2^14),
    binary16 overflow of a scaled product, subnormal scaled Gaussians): the
    flagged paths are replayed in the emulation, so the moments still equal
    the dump kernel's per-path values reduced by the restated tree."""
    n = 4000
    model = gpu.make_gbm(mu, sigma, x0, 1.0)
    tb = gpu.InvCdfApprox.parse("linear:16")
    if not gpu.api.bar_arithmetic(model, level, fp16(gpu), tb, kahan)["native_binary16"]:
        pytest.skip("the host keeps this model on the emulation")
    out, want = _want(gpu, oracle, model, level, tb, n, 3, level << 40, kahan=kahan)
    cfg = oracle.config(level=level, mantissa_bits=10, approx="linear:16", kahan=kahan, seed=3,
                        mu=mu, sigma=sigma, x0=x0)
    own, _, fails = oracle.simulate(cfg, level << 40, n)
    assert not fails
    assert np.array_equal(bits(out[:, 2:]), bits(own[:, 2:]))
    assert _moments(gpu, model, level, tb, n, 3, level << 40, kahan) == want


@pytest.mark.gpu
@pytest.mark.parametrize("kahan", [False, True])
def test_native_binary16_full_chunk(gpu, oracle, kahan):
    """A whole 2^18-path chunk at level 8 (the persistent kernel's three
    groups over 1024 batches): moments of the native run equal the dump
    kernel's values reduced by the restated tree."""
    n, level = 262144 + 300, 8
    model = gpu.make_gbm()
    tb = gpu.InvCdfApprox.parse("linear:16")
    out, want = _want(gpu, oracle, model, level, tb, n, 1, level << 40, "all", "call", kahan)
    assert _moments(gpu, model, level, tb, n, 1, level << 40, kahan, legs="all", payoff="call",
                    strike=1.0) == want
