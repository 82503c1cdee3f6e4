"""Throughput of the BASELINE.json configurations other than the bench's own
(C2), one GPU, device-timed with CUDA events around plan launches.

    python tools/bench_configs.py [--quick] > profiles/r01_configs.json

C1  level 6, fp64 exact, 2-way hat legs only (and all four legs), 2^20 paths;
    also in LPMC_EXACT_Z_GLIBC mode (the reference's Z bit for bit), with the
    C2 level-10 launch
C3  fp16 bar legs (native IEEE half2 and the emulated m=10 reference
    arithmetic), constant:16 / linear:16, +-Kahan, levels 0..8, 2^24 paths,
    bar legs only
C4  4-way call payoff max(S-1, 0), exact fp64 + approx fp32 / fp16 (emulated),
    linear:16, levels 0..12, 2^24 paths
C5  sample of the sweep: level 14, 2^24 paths (the full 2^30 x 15 levels x
    6 variants is ~2e14 path-steps per GPU), fp32 +-Kahan and fp16, 2-way and
    4-way (all legs)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2012_09739_b200 as L  # noqa: E402


def timed(plan, stream, reps=3):
    plan.launch(stream.cuda_stream)
    plan.collect()
    best = None
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        plan.launch(stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
        plan.collect()
    return best


def run(name, level, spec, approx, kahan, n, legs="all", payoff="terminal", stream=None,
        exact_z="fast"):
    plan = L.LevelPlan(L.make_gbm(), level, spec, approx, kahan, n, 1, level << 40, legs=legs,
                       payoff=payoff, strike=1.0, exact_z=exact_z)
    ms = timed(plan, stream)
    m = plan.collect() if False else None  # noqa: F841
    plan.launch(stream.cuda_stream)
    res = plan.collect()
    plan.close()
    steps = n << level
    return {"config": name, "level": level, "mantissa_bits": spec.mantissa_bits,
            "ieee_half": spec.ieee_half, "approx": None if approx is None else approx.kind + ":" +
            str(approx.interval_count()), "kahan": kahan, "legs": legs, "payoff": payoff,
            "exact_z": exact_z,
            "paths": n, "ms": ms, "path_steps_per_s": steps / (ms * 1e-3),
            "v_hat": res.d_hat.variance(), "v_bar": res.d_bar.variance(),
            "V_bar": res.d_four.variance()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    lin = L.InvCdfApprox.parse("linear:16")
    con = L.InvCdfApprox.parse("constant:16")
    P = L.PrecisionSpec
    out = []
    n20, n24 = 1 << 20, 1 << 24
    if a.quick:
        n24 = 1 << 22
    out.append(run("C1", 6, P.carrier(), None, False, n20, legs="hat", stream=s))
    out.append(run("C1-all-legs", 6, P.carrier(), None, False, n20, stream=s))
    # the reference's Z bit for bit (LPMC_EXACT_Z_GLIBC): C1 and the C2 level 10
    out.append(run("C1-glibc", 6, P.carrier(), None, False, n20, legs="hat", stream=s,
                   exact_z="glibc"))
    out.append(run("C2-l10-glibc", 10, P.fp32(), lin, False, 1 << 22, stream=s, exact_z="glibc"))
    for spec, tag in ((P.fp16_ieee(), "C3-ieee-half2"), (P.fp16(), "C3-emulated-m10")):
        for tab in (con, lin):
            for k in (False, True):
                for level in (0, 4, 8):
                    out.append(run(tag, level, spec, tab, k, n24, legs="bar", stream=s))
    for spec, tag in ((P.fp32(), "C4-fp32"), (P.fp16(), "C4-fp16-emulated")):
        for level in (0, 6, 12):
            out.append(run(tag, level, spec, lin, False, n24, payoff="call", stream=s))
    for spec, k, tag in ((P.fp32(), False, "C5-fp32"), (P.fp32(), True, "C5-fp32-kahan"),
                         (P.fp16(), False, "C5-fp16-emulated"),
                         (P.fp16_ieee(), False, "C5-fp16-ieee")):
        out.append(run(tag, 14, spec, lin, k, 1 << 22 if a.quick else n24, stream=s))
        out.append(run(tag + "-2way-bar", 14, spec, lin, k, 1 << 22 if a.quick else n24,
                       legs="bar", stream=s))
    json.dump({"device": torch.cuda.get_device_name(0), "results": out}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
