"""Stress check of the native binary16 / bfloat16 legs against the
fp32-carried emulation (the same build, LPMC_NO_NATIVE_HALF / _BF16): the
production moments of both must be identical bit for bit -- many seeds,
levels 0..14, +-Kahan, all / bar / fine legs, 2^20 paths per run (about 1e13
path-steps in total); then the power-of-two folded kernels against the
unfolded ones (LPMC_NO_POW2) for every bar arithmetic and the hat-only
instances.

    python tools/stress_native.py [runs_per_precision]
"""
from __future__ import annotations

import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2012_09739_b200 as L  # noqa: E402


def moments(model, level, spec, tb, kahan, n, seed, base, **ext):
    m = L.run_coupled_paths(model, level, spec, tb, kahan, n, seed, base, **ext)
    return [m.d_hat.state(), m.d_bar.state(), m.d_four.state()]


def main():
    runs = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    rng = np.random.default_rng(20260101)
    tables = [L.InvCdfApprox.parse("linear:16"), L.InvCdfApprox.parse("linear:8"), None]
    bad = 0
    steps = 0
    t0 = time.time()
    for name, spec, env in (("fp16", L.PrecisionSpec(10, False), "LPMC_NO_NATIVE_HALF"),
                            ("bf16", L.PrecisionSpec(7, False), "LPMC_NO_NATIVE_BF16")):
        for i in range(runs):
            level = int(rng.integers(0, 15))
            kahan = bool(rng.integers(0, 2))
            legs = ["all", "bar", "fine"][int(rng.integers(0, 3))]
            tb = tables[int(rng.integers(0, 3))]
            seed = int(rng.integers(1, 1 << 40))
            base = int(rng.integers(0, 1 << 44))
            n = 1 << 20 if level <= 12 else 1 << 18
            sigma = [0.2, 0.2, 0.4, 0.1, 1.5][int(rng.integers(0, 5))]
            mu = [0.05, 0.05, -0.1, 0.3][int(rng.integers(0, 4))]
            x0 = [1.0, 1.0, 0.5, 3.0, 0.125, 100.0][int(rng.integers(0, 6))]
            model = L.make_gbm(mu, sigma, x0, 1.0)
            ext = {"legs": legs, "payoff": "call" if i % 2 else "terminal", "strike": 1.0}
            got = moments(model, level, spec, tb, kahan, n, seed, base, **ext)
            os.environ[env] = "1"
            try:
                want = moments(model, level, spec, tb, kahan, n, seed, base, **ext)
            finally:
                del os.environ[env]
            steps += 2 * (n << level)
            if got != want:
                bad += 1
                print(f"MISMATCH {name} level {level} kahan {kahan} legs {legs} "
                      f"table {tb is not None} seed {seed} base {base} mu {mu} sigma {sigma} x0 {x0}")
    # power-of-two step folding (step_hat_pw, step_bar_pw) against the unfolded
    # kernels (LPMC_NO_POW2), even levels, every bar arithmetic
    folded = 0
    specs = [("fp32", L.PrecisionSpec.fp32()), ("fp64", L.PrecisionSpec(52, False)),
             ("fp16", L.PrecisionSpec(10, False)), ("bf16", L.PrecisionSpec(7, False))]
    for i in range(runs):
        name, spec = specs[int(rng.integers(0, 4))]
        level = 2 * int(rng.integers(0, 8))
        kahan = bool(rng.integers(0, 2))
        legs = ["all", "bar", "fine", "hat"][int(rng.integers(0, 4))]
        tb = tables[int(rng.integers(0, 3))]
        if legs == "hat":
            tb, kahan, spec = None, False, L.PrecisionSpec(52, False)
        seed = int(rng.integers(1, 1 << 40))
        base = int(rng.integers(0, 1 << 44))
        n = 1 << 20 if level <= 12 else 1 << 18
        sigma = [0.2, 0.4, 0.1, 1.5][int(rng.integers(0, 4))]
        mu = [0.05, -0.1, 0.3][int(rng.integers(0, 3))]
        model = L.make_gbm(mu, sigma, [1.0, 0.5, 3.0][int(rng.integers(0, 3))], 1.0)
        ext = {"legs": legs, "payoff": "call" if i % 2 else "terminal", "strike": 1.0}
        if not L.api.bar_arithmetic(model, level, spec, tb, kahan, legs=legs)["pow2_folded"]:
            continue
        folded += 1
        got = moments(model, level, spec, tb, kahan, n, seed, base, **ext)
        os.environ["LPMC_NO_POW2"] = "1"
        try:
            assert not L.api.bar_arithmetic(model, level, spec, tb, kahan,
                                            legs=legs)["pow2_folded"]
            want = moments(model, level, spec, tb, kahan, n, seed, base, **ext)
        finally:
            del os.environ["LPMC_NO_POW2"]
        steps += 2 * (n << level)
        if got != want:
            bad += 1
            print(f"MISMATCH folded {name} level {level} kahan {kahan} legs {legs} "
                  f"table {tb is not None} seed {seed} base {base} mu {mu} sigma {sigma}")
    print(f"stress: {2 * runs} native/emulated and {folded} folded/unfolded run pairs, "
          f"{steps:.3e} path-steps, {bad} mismatches, {time.time() - t0:.1f} s")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
