"""Measurement of the callers above the level sampler (SURVEY.md §8f rows
1-3) on one GPU, each beside the unmodified reference on the host's cores
(oracle/_ref, threads = all cores where the reference takes a thread count).

    python tools/bench_callers.py > profiles/r01_callers.json

Every timing is end to end through the public API (host arguments in, host
results out), best of 3 after one warm-up, wall clock with the device
synchronised by the blocking call itself.
  nested      run_nested_estimator, fp16 (emulated) linear:16, levels 0..8
  two_way     run_two_way_experiment, fp16 linear:1024, levels 0..12, the
              reference's default path counts (1e4, halved above level 9)
  four_way    run_four_way_experiment, fp16/fp32 linear:16, levels 0..10, 2e4 paths
  probe       step_error_probe, fp16 linear:16, level 10, 1e7 samples
  density     run_density_report, reference defaults (linear:1024, 2047 curve
              points, 1e6 histogram samples, bin width 0.05), and exact
  concurrency the nested estimator's pilot pass (11 levels x 1000 paths):
              one run_coupled_many call vs 11 run_coupled_paths calls
Throughput unit: fine path-steps (paths x 2^level, summed) per second.
"""
from __future__ import annotations

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2012_09739_b200 as L  # noqa: E402
from oracle.bind import Reference  # noqa: E402
from paper_2012_09739_b200.experiments import (ExperimentConfig,  # noqa: E402
                                               run_density_report, run_four_way_experiment,
                                               run_two_way_experiment)


def best_of(fn, reps=3):
    fn()
    best = None
    for _ in range(reps):
        t = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return best, out


def once(fn):
    t = time.perf_counter()
    out = fn()
    return time.perf_counter() - t, out


def main():
    R = Reference()
    cores = R.hardware_threads()
    res = {"device": None, "host_threads": cores, "results": []}
    import torch
    res["device"] = torch.cuda.get_device_name(0)
    model = L.make_gbm()

    # ---- nested estimator
    lin16 = L.InvCdfApprox.parse("linear:16")
    for max_level, eps in ((8, 2e-4), (4, 1e-4)):
        t_gpu, r = best_of(lambda: L.run_nested_estimator(model, max_level, L.PrecisionSpec.fp16(),
                                                          lin16, False, eps, 1))
        steps = sum(1000 << l for l in range(max_level + 1)) + sum(
            (p + s) << l for l, (p, s) in enumerate(zip(r.allocation.primary,
                                                        r.allocation.secondary)))
        t_cpu, (rc, msg, rr) = once(lambda: R.run_nested_estimator(
            max_level=max_level, mantissa_bits=10, approx="linear:16", eps=eps, threads=cores))
        assert rc == 0, msg
        res["results"].append({
            "row": "nested_estimator", "max_level": max_level, "eps": eps, "precision": "fp16",
            "approx": "linear:16", "fine_path_steps": steps, "gpu_s": t_gpu, "ref_cpu_s": t_cpu,
            "speedup": t_cpu / t_gpu, "gpu_path_steps_per_s": steps / t_gpu,
            "ref_path_steps_per_s": steps / t_cpu, "value_gpu": r.value, "value_ref": rr["value"],
            "allocation_equal": r.allocation.primary == rr["primary"] and
            r.allocation.secondary == rr["secondary"]})

    # ---- two-way experiment (reference defaults)
    cfg = ExperimentConfig(precisions=["fp16"], approx="linear:1024", level_min=0, level_max=12)
    steps = sum(cfg.paths_for_level(l) << l for l in range(13))
    t_gpu, rows = best_of(lambda: run_two_way_experiment(cfg))
    t_cpu, (rc, msg, out) = once(lambda: R.two_way_experiment(
        precision="fp16", approx="linear:1024", kahan=0, level_min=0, level_max=12, paths=0,
        threads=cores))
    assert rc == 0, msg
    res["results"].append({"row": "two_way_experiment", "levels": "0..12", "paths": "default",
                           "fine_path_steps": steps, "gpu_s": t_gpu, "ref_cpu_s": t_cpu,
                           "speedup": t_cpu / t_gpu, "gpu_path_steps_per_s": steps / t_gpu,
                           "max_rel_variance_diff": max(abs(g.variance - w[1]) / w[1]
                                                        for g, w in zip(rows, out))})

    # ---- four-way experiment (GPU only + per-level reference sample)
    cfg4 = ExperimentConfig(precisions=["fp16", "fp32"], approx="linear:16", level_min=0,
                            level_max=10, paths=[20000])
    steps4 = 3 * sum(20000 << l for l in range(11))
    t_gpu4, _ = best_of(lambda: run_four_way_experiment(cfg4))
    t_cpu4 = 0.0
    for l in range(11):
        for m, k, ph in ((10, 0, 0), (10, 1, 1), (23, 0, 2)):
            dt, (rc, msg, _) = once(lambda: R.estimate_level_stats(
                level=l, mantissa_bits=m, approx="linear:16", kahan=k, n=20000, threads=cores,
                path_base=(l << 40) | (ph << 36)))
            assert rc == 0, msg
            t_cpu4 += dt
    res["results"].append({"row": "four_way_experiment", "levels": "0..10", "paths": 20000,
                           "fine_path_steps": steps4, "gpu_s": t_gpu4, "ref_cpu_s": t_cpu4,
                           "speedup": t_cpu4 / t_gpu4, "gpu_path_steps_per_s": steps4 / t_gpu4,
                           "ref_path_steps_per_s": steps4 / t_cpu4})

    # ---- step-error probe
    n = 10_000_000
    t_gpu, st = best_of(lambda: L.step_error_probe(model, 10, L.PrecisionSpec.fp16(), lin16, n, 1))
    t_cpu, (rc, msg, out) = once(lambda: R.step_error_probe(level=10, mantissa_bits=10,
                                                             approx="linear:16", n_samples=n))
    assert rc == 0, msg
    res["results"].append({"row": "step_error_probe", "level": 10, "samples": n,
                           "gpu_s": t_gpu, "ref_cpu_s": t_cpu, "ref_threads": 1,
                           "speedup": t_cpu / t_gpu, "gpu_steps_per_s": n / t_gpu,
                           "rel_diff_mean_abs_eta": abs(st.mean_abs_eta - out[1]) / out[1]})

    # ---- density report
    for approx in ("linear:1024", "exact"):
        cfgd = ExperimentConfig(approx=approx, level_min=0, level_max=0)
        t_gpu, rows = best_of(lambda: run_density_report(cfgd))
        t_cpu, (rc, msg, out) = once(lambda: R.density_report(approx=approx))
        assert rc == 0, msg
        same = sum(1 for r, w in zip(rows, out) if r.y == w[2])
        res["results"].append({"row": "density_report", "approx": approx, "samples": 1000000,
                               "gpu_s": t_gpu, "ref_cpu_s": t_cpu, "ref_threads": 1,
                               "speedup": t_cpu / t_gpu, "rows": len(rows),
                               "rows_bitwise_equal": same})

    # ---- concurrency of the multi-run entry point
    runs = [(l, L.PrecisionSpec.fp16(), False, 1000, l << 40) for l in range(11)]
    t_many, _ = best_of(lambda: L.run_coupled_many(model, lin16, 1, runs))
    t_loop, _ = best_of(lambda: [L.run_coupled_paths(model, l, s, lin16, k, n_, 1, b)
                                 for l, s, k, n_, b in runs])
    res["results"].append({"row": "run_coupled_many_pilot", "runs": 11, "paths_per_run": 1000,
                           "many_s": t_many, "serial_loop_s": t_loop,
                           "speedup": t_loop / t_many})
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
