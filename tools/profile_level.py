"""One level launch of the sampler, for ncu (-k regex:level_kernel -s 1 -c 1).

    python tools/profile_level.py --level 10 --prec fp32 --approx linear:16
Launch 0 warms up, launch 1 is the profiled one; both are the C2 level config.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2012_09739_b200 as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=10)
    ap.add_argument("--prec", default="fp32")
    ap.add_argument("--approx", default="linear:16")
    ap.add_argument("--kahan", type=int, default=0)
    ap.add_argument("--legs", default="all")
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--launches", type=int, default=2)
    ap.add_argument("--payoff", default="terminal", choices=["terminal", "call"])
    ap.add_argument("--base", type=int, default=None, help="path base (default level<<40 | kahan<<36)")
    ap.add_argument("--exact-z", default="fast", choices=["fast", "glibc"])
    ap.add_argument("--schedule", default="auto", choices=["auto", "fused", "warp_per_path"])
    ap.add_argument("--time", action="store_true",
                    help="also time 5 launches with CUDA events (best of, ms)")
    a = ap.parse_args()
    spec = L.PrecisionSpec.parse(a.prec)
    approx = None if a.approx == "exact" else L.InvCdfApprox.parse(a.approx)
    plan = L.LevelPlan(L.make_gbm(), a.level, spec, approx, bool(a.kahan), a.n, 1,
                       (a.level << 40) | (a.kahan << 36) if a.base is None else a.base,
                       legs=a.legs, exact_z=a.exact_z, schedule=a.schedule, payoff=a.payoff,
                       strike=1.0)
    for _ in range(a.launches):
        plan.launch()
        m = plan.collect()
    print(f"level {a.level} {a.prec} {a.approx} kahan={a.kahan} legs={a.legs} n={a.n} "
          f"exact_z={a.exact_z}: "
          f"v_hat={m.d_hat.variance():.6e} v_bar={m.d_bar.variance():.6e} "
          f"V_bar={m.d_four.variance():.6e}")
    if a.time:
        import torch
        st = torch.cuda.Stream()
        best = None
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            plan.launch(st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            plan.collect()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        print(f"time_ms {best:.4f} path_steps_per_s {(a.n << a.level) / (best * 1e-3):.4e}")
    plan.close()


if __name__ == "__main__":
    main()
