"""The hot loop's special-draw prefilter (lpmc_level.cuh draw_uniforms,
DESIGN.md section 8 "Special-draw prefilter").

The unchecked level kernel flags a path for the exact replay when a draw
b = w >> 11 has a low word of 0 or 0xffffffff: a superset of the two special
draws (b = 2^52, u == 1/2; b = 2^53 - 1, u == 1).  These tests build seeds
whose stream hits such a low word on an ordinary draw (by inverting mix64,
uniform.hpp:13-27), check the construction against the oracle's stream, and
check on the device that the false-positive path's four legs and the
level's moments equal the oracle's bitwise.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import bits

M64 = (1 << 64) - 1
C1, C2 = 0xFF51AFD7ED558CCD, 0xC4CEB9FE1A85EC53
PHI, PATH_C, CTR_C = 0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9, 0x94D049BB133111EB
HALF_DRAW, TOP_DRAW = 1 << 52, (1 << 53) - 1


def mix64(z: int) -> int:  # uniform.hpp:13-20
    z ^= z >> 33
    z = (z * C1) & M64
    z ^= z >> 33
    z = (z * C2) & M64
    z ^= z >> 33
    return z


def unmix64(z: int) -> int:
    # z ^= z >> 33 is an involution for a shift >= 32; odd multipliers invert mod 2^64
    z ^= z >> 33
    z = (z * pow(C2, -1, 1 << 64)) & M64
    z ^= z >> 33
    z = (z * pow(C1, -1, 1 << 64)) & M64
    z ^= z >> 33
    return z


def stream_draw(seed: int, path: int, ctr: int) -> int:  # uniform.hpp:22-27, b = w >> 11
    key = mix64(mix64((seed + PHI) & M64) ^ mix64((path + PATH_C) & M64))
    return mix64(mix64((key + ctr * CTR_C) & M64)) >> 11


def seed_for_draw(b: int, path: int, ctr: int) -> int:
    """A seed whose stream for `path` draws exactly b at counter `ctr`."""
    key = (unmix64(unmix64(b << 11)) - ctr * CTR_C) & M64
    return (unmix64(unmix64(key) ^ mix64((path + PATH_C) & M64)) - PHI) & M64


# ordinary draws whose low word trips the prefilter (u ~ 2.3e-6 and ~ 0.78)
CASES = [((5 << 32), 17, 9), ((0x18F3A7 << 32) | 0xFFFFFFFF, 131, 2)]


@pytest.mark.parametrize("b,path,ctr", CASES)
def test_constructed_seed_hits_the_draw(oracle, b, path, ctr):
    assert b not in (HALF_DRAW, TOP_DRAW) and (b & 0xFFFFFFFF) in (0, 0xFFFFFFFF)
    seed = seed_for_draw(b, path, ctr)
    assert stream_draw(seed, path, ctr) == b
    # the same draw through the oracle's restated stream (pinned against the reference)
    u = oracle.uniforms(seed, path, 1, ctr)[0]
    assert u == b * 2.0 ** -53 + 2.0 ** -54
    # both special draws have the low words the prefilter tests
    assert HALF_DRAW & 0xFFFFFFFF == 0 and TOP_DRAW & 0xFFFFFFFF == 0xFFFFFFFF


@pytest.mark.gpu
@pytest.mark.parametrize("b,path,ctr", CASES)
@pytest.mark.parametrize("m,approx,kahan", [(23, "linear:16", False), (10, "cubic:64", True),
                                             (52, "exact", False)])
def test_false_positive_path_is_exact(gpu, oracle, b, path, ctr, m, approx, kahan):
    level, base, n = 4, 1000, 300  # fused schedule (warp-per-path only from level 5)
    seed = seed_for_draw(b, base + path, ctr)
    model = gpu.make_gbm()
    sp = gpu.PrecisionSpec(m, False)
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    out, z = gpu.simulate_paths(model, level, sp, tb, kahan, n, seed, base, want_z=True)
    cfg = oracle.config(level=level, mantissa_bits=m, approx=approx, kahan=kahan, seed=seed)
    rep, _, fails = oracle.simulate(cfg, base, n, z_in=z)
    assert not fails
    assert np.array_equal(bits(out), bits(rep))  # all four legs, incl. the flagged path
    if approx != "exact":  # bar legs need no libm: bitwise the oracle's own run
        own, _, _ = oracle.simulate(cfg, base, n)
        assert np.array_equal(bits(out[:, 2:]), bits(own[:, 2:]))
    dh = out[:, 0] - out[:, 1]
    db = out[:, 2] - out[:, 3]
    got = gpu.run_coupled_paths(model, level, sp, tb, kahan, n, seed, base)
    assert [got.d_hat.state(), got.d_bar.state(), got.d_four.state()] == \
        oracle.tree_from_values(dh, db)


# ---- the two genuinely special draws mid-path ----------------
# u == 1/2 (b = 2^52): both transforms return exactly +0 (gaussian.hpp:62,
# invcdf_approx.hpp:47); the prefilter sends the path to the exact replay,
# whose legs and dumped Gaussians must be the oracle's bitwise.
# u == 1 (b = 2^53 - 1): the reference throws domain_error("exact_inv_cdf
# requires u in (0, 1)") at that draw; the device reports the same exception
# with the path index and the step.
SPECIAL_PRECS = [(23, False, "linear:16", False), (10, False, "cubic:64", True),
                 (52, False, "exact", False), (10, True, "linear:16", False)]
SPECIAL_IDS = ["fp32-lin16", "fp16-cubic64-K", "fp64-exact", "half2-lin16"]


@pytest.mark.gpu
@pytest.mark.parametrize("exact_z", ["fast", "glibc"])
@pytest.mark.parametrize("m,ieee,approx,kahan", SPECIAL_PRECS, ids=SPECIAL_IDS)
@pytest.mark.parametrize("path,ctr", [(17, 9), (130, 0), (299, 63)])
def test_half_draw_mid_path(gpu, oracle, exact_z, m, ieee, approx, kahan, path, ctr):
    level, base, n = 6, 1000, 300
    seed = seed_for_draw(HALF_DRAW, base + path, ctr)
    assert stream_draw(seed, base + path, ctr) == HALF_DRAW
    assert oracle.uniforms(seed, base + path, 1, ctr)[0] == 0.5
    model = gpu.make_gbm()
    sp = gpu.PrecisionSpec(m, ieee)
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    ext = {"exact_z": exact_z}
    out, z = gpu.simulate_paths(model, level, sp, tb, kahan, n, seed, base, want_z=True,
                                schedule="fused", **ext)
    assert bits(z[path, ctr:ctr + 1]).tolist() == [0]  # exactly +0 in the dump
    cfg = oracle.config(level=level, mantissa_bits=m, approx=approx, kahan=kahan, seed=seed,
                        ieee_half=ieee)
    rep, _, fails = oracle.simulate(cfg, base, n, z_in=z)
    assert not fails
    assert np.array_equal(bits(out), bits(rep))
    own, zo, _ = oracle.simulate(cfg, base, n, want_z=True)
    assert zo[path, ctr] == 0.0
    if approx != "exact" or exact_z == "glibc":
        cols = slice(0, 4) if exact_z == "glibc" else slice(2, 4)
        assert np.array_equal(bits(out[:, cols]), bits(own[:, cols]))
    if not ieee:  # the warp-per-path schedule (NP == 1 arithmetics): same terminal values
        wpp = gpu.simulate_paths(model, level, sp, tb, kahan, n, seed, base,
                                 schedule="warp_per_path", **ext)
        assert np.array_equal(bits(wpp), bits(out))
    got = gpu.run_coupled_paths(model, level, sp, tb, kahan, n, seed, base, **ext)
    dh = out[:, 0] - out[:, 1]
    db = out[:, 2] - out[:, 3]
    assert [got.d_hat.state(), got.d_bar.state(), got.d_four.state()] == \
        oracle.tree_from_values(dh, db)


@pytest.mark.gpu
@pytest.mark.parametrize("exact_z", ["fast", "glibc"])
@pytest.mark.parametrize("sched", ["fused", "warp_per_path"])
@pytest.mark.parametrize("m,ieee,approx,kahan", SPECIAL_PRECS, ids=SPECIAL_IDS)
def test_top_draw_raises_at_its_step(gpu, ref, exact_z, sched, m, ieee, approx, kahan):
    level, base, n, path, ctr = 6, 1000, 300, 211, 37
    seed = seed_for_draw(TOP_DRAW, base + path, ctr)
    if ieee and sched == "warp_per_path":
        pytest.skip("half2 legs run two paths per thread (fused schedule only)")
    model = gpu.make_gbm()
    sp = gpu.PrecisionSpec(m, ieee)
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    # the reference itself throws at this draw (the same message)
    rc, msg, _ = ref.run_coupled_paths(level=level, mantissa_bits=m, approx=approx, kahan=kahan,
                                       n=n, seed=seed, path_base=base, threads=1)
    assert rc == 2 and "exact_inv_cdf requires u in (0, 1)" in msg
    for call in ("run", "dump"):
        with pytest.raises(gpu.DomainError, match=r"exact_inv_cdf requires u in \(0, 1\)") as ei:
            if call == "run":
                gpu.run_coupled_paths(model, level, sp, tb, kahan, n, seed, base, schedule=sched,
                                      exact_z=exact_z)
            else:
                gpu.simulate_paths(model, level, sp, tb, kahan, n, seed, base, schedule=sched,
                                   exact_z=exact_z)
        assert ei.value.path_index == base + path
        assert ei.value.step == ctr


# ---- the smallest draw (b = 0, u = 2^-54) ----------------------------------
# 1 - u rounds to 1, so the approximate transform's v = 1 - fl(1 - u) is 0:
# the reference maps it to the clamped tail (invcdf_approx.hpp:47-49, :61),
# the dyadic-linear device code reads its last tail record (the index of v ==
# 0 wraps; lpmc_device.cuh approx_inv).  The exact transform takes the path
# below the direct table.  Schedules, precisions and table kinds as above.
@pytest.mark.gpu
@pytest.mark.parametrize("sched", ["fused", "warp_per_path"])
@pytest.mark.parametrize("m,ieee,approx,kahan", SPECIAL_PRECS, ids=SPECIAL_IDS)
def test_bottom_draw_mid_path(gpu, oracle, sched, m, ieee, approx, kahan):
    level, base, n, path, ctr = 6, 1000, 300, 77, 21
    if ieee and sched == "warp_per_path":
        pytest.skip("half2 legs run two paths per thread (fused schedule only)")
    seed = seed_for_draw(0, base + path, ctr)
    assert stream_draw(seed, base + path, ctr) == 0
    assert oracle.uniforms(seed, base + path, 1, ctr)[0] == 2.0 ** -54
    model = gpu.make_gbm()
    sp = gpu.PrecisionSpec(m, ieee)
    tb = None if approx == "exact" else gpu.InvCdfApprox.parse(approx)
    out, z = gpu.simulate_paths(model, level, sp, tb, kahan, n, seed, base, want_z=True,
                                schedule=sched)
    cfg = oracle.config(level=level, mantissa_bits=m, approx=approx, kahan=kahan, seed=seed,
                        ieee_half=ieee)
    own, zo, fails = oracle.simulate(cfg, base, n, want_z=True)
    assert not fails
    assert abs(z[path, ctr] - zo[path, ctr]) <= 4 * 2.0 ** -52 * abs(zo[path, ctr])
    assert zo[path, ctr] < -8.0
    rep, _, _ = oracle.simulate(cfg, base, n, z_in=z)
    assert np.array_equal(bits(out), bits(rep))
    if approx != "exact":  # bar legs: the oracle's own run, incl. the tail value
        assert np.array_equal(bits(out[:, 2:]), bits(own[:, 2:]))
    got = gpu.run_coupled_paths(model, level, sp, tb, kahan, n, seed, base, schedule=sched)
    dh = out[:, 0] - out[:, 1]
    db = out[:, 2] - out[:, 3]
    assert [got.d_hat.state(), got.d_bar.state(), got.d_four.state()] == \
        oracle.tree_from_values(dh, db)
