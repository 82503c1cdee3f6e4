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


def callers():
    """Fixtures of the callers above the level sampler:
    two-way paths and experiment rows, allocation/predicted-time/speedup pins,
    nested-estimator runs -> callers_vectors.json."""
    build(ref=True)
    R = Reference()
    threads = os.cpu_count() or 1

    two_way_paths = []
    for level in [0, 1, 3, 6]:
        for m in [52, 23, 10]:
            for approx in ["exact", "linear:16", "cubic:64"]:
                for kahan in [0, 1]:
                    rc, msg, out = R.simulate_two_way(level=level, mantissa_bits=m, approx=approx,
                                                      kahan=kahan, seed=3, path_base=77 + level,
                                                      n=16)
                    assert rc == 0, msg
                    two_way_paths.append({"level": level, "m": m, "approx": approx,
                                          "kahan": kahan, "seed": 3, "path_base": 77 + level,
                                          "out": hx(out)})

    two_way_rows = []
    for prec, approx, kahan, lmin, lmax, paths in [("fp16", "linear:16", 0, 0, 6, 2000),
                                                   ("fp16", "linear:16", 1, 0, 6, 2000),
                                                   ("fp32", "cubic:64", 0, 0, 4, 3000),
                                                   ("bf16", "exact", 0, 2, 5, 1500)]:
        rc, msg, out = R.two_way_experiment(precision=prec, approx=approx, kahan=kahan,
                                            level_min=lmin, level_max=lmax, paths=paths,
                                            threads=threads)
        assert rc == 0, msg
        two_way_rows.append({"precision": prec, "approx": approx, "kahan": kahan,
                             "level_min": lmin, "level_max": lmax, "paths": paths,
                             "rows": [hx(r) for r in out]})

    rng = np.random.default_rng(11)

    def stats_set(n, zero=()):
        out = []
        for lv in range(n):
            d = {k: 0.0 for k in Reference.STATS_FIELDS}
            d.update(level=lv, v_hat=float(rng.uniform(1e-6, 1e-3)), c_hat=3.5 * 2**lv,
                     v_bar=float(rng.uniform(1e-6, 1e-3)), c_bar=0.25 * 2**lv * 1.4,
                     V_bar=float(rng.uniform(1e-9, 1e-5)))
            d["C_bar"] = d["c_hat"] + d["c_bar"]
            for k in zero:
                d[k] = 0.0
            out.append(d)
        return out

    sets = [stats_set(6), stats_set(3, zero=("v_bar",)), stats_set(4, zero=("v_hat", "v_bar",
                                                                            "V_bar")),
            stats_set(1)]
    allocation = []
    for si, st in enumerate(sets):
        for eps in [1e-3, 2.5e-2]:
            for kind in [0, 1]:
                rc, msg, (prim, sec, deg) = R.allocate_samples(st, eps, kind)
                allocation.append({"set": si, "eps": eps.hex(), "kind": kind, "rc": rc,
                                   "msg": msg, "primary": prim, "secondary": sec,
                                   "degenerate": deg})
    bad_alloc = []
    for st, eps in [([], 1e-3), (sets[0], 0.0), (sets[0], -1.0)]:
        rc, msg, _ = R.allocate_samples(st, eps, 1)
        bad_alloc.append({"n": len(st), "eps": eps.hex(), "rc": rc, "msg": msg})
    times = []
    for si, st in enumerate(sets):
        rc, msg, (th, tb) = R.predicted_times(st, 1e-3)
        times.append({"set": si, "eps": (1e-3).hex(), "rc": rc, "t_hat": th.hex(),
                      "t_bar": tb.hex()})
    speedup = []
    for si, st in enumerate(sets):
        for li, row in enumerate(st):
            rc, msg, (v, flag) = R.per_level_speedup(row)
            speedup.append({"set": si, "level": li, "rc": rc, "msg": msg, "value": v.hex(),
                            "cost_ratio_only": flag})

    nested = []
    for max_level, m, approx, kahan, eps in [(4, 10, "linear:16", 0, 1e-3),
                                             (3, 23, "linear:16", 1, 2e-3),
                                             (3, 52, "exact", 0, 5e-3),
                                             (0, 10, "linear:8", 0, 1e-2)]:
        rc, msg, r = R.run_nested_estimator(max_level=max_level, mantissa_bits=m, approx=approx,
                                            kahan=kahan, eps=eps, threads=threads)
        assert rc == 0, msg
        nested.append({"max_level": max_level, "m": m, "approx": approx, "kahan": kahan,
                       "eps": eps.hex(), "seed": 1, "pilot_paths": 1000,
                       "value": r["value"].hex(), "t_hat": r["t_hat"].hex(),
                       "t_bar": r["t_bar"].hex(), "degenerate": r["degenerate"],
                       "contributions": hx(r["contributions"]), "pilot": hx(r["pilot"]),
                       "primary": r["primary"], "secondary": r["secondary"]})
    nested_errors = []
    for max_level, eps, pilot in [(-1, 1e-3, 1000), (2, 0.0, 1000), (2, 1e-3, 1)]:
        rc, msg, _ = R.run_nested_estimator(max_level=max_level, mantissa_bits=10,
                                            approx="linear:16", eps=eps, pilot_paths=pilot)
        nested_errors.append({"max_level": max_level, "eps": eps.hex(), "pilot_paths": pilot,
                              "rc": rc, "msg": msg})

    probe = []
    for level, m, approx, n_samples, seed in [(0, 10, "linear:16", 100000, 1),
                                              (3, 23, "linear:16", 100000, 2),
                                              (6, 7, "cubic:64", 65536 + 123, 3),
                                              (10, 10, "exact", 50000, 1),
                                              (2, 52, "linear:16", 10000, 4),
                                              (4, 23, "exact", 100000, 5),
                                              (12, 16, "linear:1024", 10000, 6),
                                              (5, 10, "linear:16", 0, 1)]:
        rc, msg, out = R.step_error_probe(level=level, mantissa_bits=m, approx=approx,
                                          n_samples=n_samples, seed=seed)
        assert rc == 0, msg
        probe.append({"level": level, "m": m, "approx": approx, "n_samples": n_samples,
                      "seed": seed, "out": hx(out)})

    density = []
    for approx, curve_points, hist, width, seed in [("linear:16", 2048, 100000, 0.05, 1),
                                                    ("cubic:64", 512, 50000, 0.1, 2),
                                                    ("linear:1024", 256, 100000, 0.05, 3),
                                                    ("exact", 2048, 100000, 0.05, 1)]:
        rc, msg, rows = R.density_report(approx=approx, seed=seed, curve_points=curve_points,
                                         hist_samples=hist, bin_width=width)
        assert rc == 0, msg
        density.append({"approx": approx, "seed": seed, "curve_points": curve_points,
                        "hist_samples": hist, "bin_width": width.hex(),
                        "rows": [[int(r[0]), float(r[1]).hex(), float(r[2]).hex()] for r in rows]})

    doc = {"generator": "tests/golden/gen_golden.py callers (reference: "
                        "/root/reference/proj/include, oracle/ref_driver.cpp)",
           "stats_fields": list(Reference.STATS_FIELDS),
           "stats_sets": [[{k: float(v).hex() for k, v in d.items()} for d in st] for st in sets],
           "two_way_paths": two_way_paths, "two_way_rows": two_way_rows,
           "allocation": allocation, "allocation_errors": bad_alloc, "times": times,
           "speedup": speedup, "nested": nested, "nested_errors": nested_errors,
           "step_error": probe, "density": density}
    with open(os.path.join(OUT, "callers_vectors.json"), "w") as f:
        json.dump(doc, f, indent=0)
    print("wrote", os.path.join(OUT, "callers_vectors.json"))


if __name__ == "__main__":
    if sys.argv[1:] == ["callers"]:
        callers()
    else:
        main()
        callers()
