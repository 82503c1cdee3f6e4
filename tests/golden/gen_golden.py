"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref).

Run here (the container that has /root/reference):

    python tests/golden/gen_golden.py

Every double is stored as float.hex() so the fixtures are bit-exact.  The
fixtures are small and committed; the GPU box never needs the reference.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.bind import Reference, build  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def hx(a):
    return [float(v).hex() for v in np.asarray(a, dtype=np.float64).reshape(-1)]


def main():
    build(ref=True)
    R = Reference()

    # a1: counter RNG (uniform.hpp:13-41)
    rng = {"words": [], "uniforms": []}
    for seed, path, ctr in [(1, 0, 0), (1, 0, 1), (42, 7, 99), (2**63 + 5, 2**40 + 3, 12345),
                            (0, 0, 0), (2**64 - 1, 2**64 - 1, 2**64 - 1)]:
        rng["words"].append([seed, path, ctr, R.stream_word(seed, path, ctr)])
    for seed, path in [(1, 0), (5, 3), (9, 2**41)]:
        rng["uniforms"].append({"seed": seed, "path": path, "u": hx(R.uniforms(seed, path, 64))})

    # a2: exact inverse CDF (gaussian.hpp:59-65), incl. both tails and u=1/2
    u = np.concatenate([R.uniforms(5, 0, 2000), [0.5, 0.02425, 0.02425 - 2**-60, 1 - 0.02425,
                                                 2**-54, 1 - 2**-53, 0.975, 1e-300]])
    gauss = {"u": hx(u), "z": hx(R.exact_inv_cdf(u))}

    # a3: tables + evaluation (invcdf_approx.hpp:44-145)
    uu = np.concatenate([R.uniforms(17, 0, 1500), [0.5, 0.75, 0.25, 1 - 2**-17, 2**-17,
                                                   1 - 2**-18, 2**-18, 1 - 2**-53, 2**-54]])
    tables = {}
    for name in ["linear:2", "linear:8", "linear:16", "linear:32", "cubic:16", "linear:64",
                 "cubic:64", "linear:1024"]:
        t = R.table(name)
        tables[name] = {"K": t.K, "w_max": t.w_max.hex(), "step_w": t.step_w.hex(),
                        "tail": t.tail.hex(), "bp": hx(t.bp), "coeff": hx(t.coeff),
                        "z": hx(R.approx(name, uu))}
    tables_u = hx(uu)

    # a4: round_to_precision (softfloat.hpp:69-80)
    x = np.concatenate([np.random.default_rng(3).standard_normal(500) * 4,
                        [1.0 + 2**-11, 1.0 + 3 * 2**-11, 1.0 + 2**-12, -1.5 - 2**-24, 0.0, -0.0,
                         1e-300, 3e300]])
    rounding = {"x": hx(x), "by_m": {str(m): hx(R.round(x, m)) for m in
                                      [1, 3, 7, 10, 16, 23, 26, 52]}}

    # a7: simulate_coupled terminal values (sde.hpp:211-284)
    paths = []
    for level in [0, 1, 2, 3, 6, 10]:
        for m in [52, 23, 10, 7, 16]:
            for approx in ["exact", "linear:16", "cubic:64"]:
                for kahan in [0, 1]:
                    if level == 10 and (m in (7, 16) or approx == "cubic:64"):
                        continue
                    n = 16 if level < 10 else 4
                    rc, msg, out = R.simulate(level=level, mantissa_bits=m, approx=approx,
                                              kahan=kahan, seed=7, path_base=1000 + level, n=n)
                    assert rc == 0, msg
                    paths.append({"level": level, "m": m, "approx": approx, "kahan": kahan,
                                  "seed": 7, "path_base": 1000 + level, "out": hx(out)})
    # reference unit-test pins (test_sde.cpp:98-128): degenerate coupling, level-1 coarse
    for level in [1, 3, 6]:
        rc, msg, out = R.simulate(level=level, mantissa_bits=52, seed=21, path_base=5, n=1)
        paths.append({"level": level, "m": 52, "approx": "exact", "kahan": 0, "seed": 21,
                      "path_base": 5, "out": hx(out)})

    # a8-a10: level moments (mlmc.hpp:67-149); raw accumulator states
    moments = []
    for level, m, approx, kahan, n, seed, base in [
        (6, 52, "exact", 0, 1 << 20, 1, 0),      # BASELINE config 1, full size
        (0, 23, "linear:16", 0, 4096, 1, 0),
        (3, 23, "linear:16", 1, 3000, 1, 3 << 40),
        (4, 10, "linear:64", 0, 1000, 5, 0),     # test_mlmc.cpp:191-202 shape
        (5, 10, "linear:16", 1, 2000, 11, (5 << 40) | (1 << 36)),
        (7, 7, "cubic:64", 0, 777, 2, 123),
        (2, 16, "exact", 1, 513, 4, 9),
        (8, 23, "linear:16", 0, 1 << 12, 1, 8 << 40),
    ]:
        rc, msg, mom = R.run_coupled_paths(level=level, mantissa_bits=m, approx=approx,
                                           kahan=kahan, n=n, seed=seed, path_base=base,
                                           threads=os.cpu_count() or 1)
        assert rc == 0, msg
        moments.append({"level": level, "m": m, "approx": approx, "kahan": kahan, "n": n,
                        "seed": seed, "path_base": base,
                        "acc": [[a[0]] + hx(a[1:]) for a in mom]})

    # error contract (sde.hpp:215, mlmc.hpp:121, softfloat.hpp:70)
    errors = []
    rc, msg, _ = R.estimate_level_stats(level=3, mantissa_bits=52, n=1)
    errors.append({"call": "estimate_level_stats", "n": 1, "level": 3, "rc": rc, "msg": msg})
    rc, msg, _ = R.run_coupled_paths(level=-1, mantissa_bits=52, n=4)
    errors.append({"call": "run_coupled_paths", "n": 4, "level": -1, "rc": rc, "msg": msg})
    rc, msg, _ = R.run_coupled_paths(level=-1, mantissa_bits=52, n=0)
    errors.append({"call": "run_coupled_paths", "n": 0, "level": -1, "rc": rc, "msg": msg})
    rc, msg, _ = R.run_coupled_paths(level=4, mantissa_bits=52, n=8, mu=1e30, sigma=0.0,
                                     x0=1e300)
    errors.append({"call": "run_coupled_paths", "n": 8, "level": 4, "mu": 1e30, "sigma": 0.0,
                   "x0": 1e300, "rc": rc, "msg": msg})

    stats = []
    for level, m, approx, kahan, n, psa in [(3, 52, "exact", 0, 64, 0.25),
                                            (0, 10, "exact", 1, 64, 0.25),
                                            (5, 23, "linear:16", 1, 2048, 0.0)]:
        rc, msg, out = R.estimate_level_stats(level=level, mantissa_bits=m, approx=approx,
                                              kahan=kahan, n=n, per_step_arithmetic=psa)
        assert rc == 0, msg
        stats.append({"level": level, "m": m, "approx": approx, "kahan": kahan, "n": n,
                      "per_step_arithmetic": psa, "out": hx(out)})

    doc = {"generator": "tests/golden/gen_golden.py (reference: /root/reference/proj/include, "
                        "oracle/ref_driver.cpp, g++ -O2 -DNDEBUG -ffp-contract=off)",
           "rng": rng, "gauss": gauss, "tables": tables, "tables_u": tables_u, "rounding": rounding,
           "paths": paths, "moments": moments, "errors": errors, "level_stats": stats}
    with open(os.path.join(OUT, "reference_vectors.json"), "w") as f:
        json.dump(doc, f, indent=0)
    print("wrote", os.path.join(OUT, "reference_vectors.json"))


if __name__ == "__main__":
    main()
