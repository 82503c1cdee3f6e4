"""Small launches of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck) on the B200:

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py

Covers: the fused level kernel (level 0 and a ragged multi-batch level, both
reductions; the shared-memory batch tree and the chunk Pebay tree), the
sequential batch kernel, the warp-per-path kernel + path_batch_kernel, the
half2 instance, glibc mode, the failure path (atomicMin on the failure key,
a u == 1 draw constructed by inverting the stream), the step-error probe and
the density histogram (shared-memory bins + atomics), the multi-run call.
"""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import paper_2012_09739_b200 as L  # noqa: E402
from test_special_prefilter import TOP_DRAW, seed_for_draw  # noqa: E402


def main():
    m = L.make_gbm()
    P = L.PrecisionSpec
    lin = L.InvCdfApprox.parse("linear:16")
    cub = L.InvCdfApprox.parse("cubic:64")
    done = []
    L.run_coupled_paths(m, 0, P.fp32(), lin, False, 1000, 1, 0)
    done.append("level 0 fused tree")
    L.run_coupled_paths(m, 3, P.fp16(), cub, True, 262144 + 777, 1, 3 << 40)
    done.append("level 3 fused tree, 2 chunks ragged")
    L.run_coupled_paths(m, 3, P.fp32(), lin, True, 3000, 1, 0, reduce="sequential")
    done.append("sequential batches")
    L.run_coupled_paths(m, 7, P.fp16(), lin, False, 300, 1, 0, schedule="warp_per_path")
    done.append("warp per path")
    L.run_coupled_paths(m, 4, P.fp16_ieee(), lin, True, 2000, 1, 0, legs="bar")
    done.append("half2 bar")
    L.run_coupled_paths(m, 4, P.fp32(), lin, False, 2000, 1, 0, exact_z="glibc", payoff="call")
    done.append("glibc mode, call payoff")
    L.run_two_way_paths(m, 5, P.fp16(), lin, True, 3000, 1, 0)
    done.append("two-way")
    seed = seed_for_draw(TOP_DRAW, 1000 + 211, 37)
    try:
        L.run_coupled_paths(m, 6, P.fp32(), lin, False, 300, seed, 1000)
    except L.DomainError as e:
        assert e.path_index == 1211 and e.step == 37
        done.append("failure replay + atomicMin")
    L.step_error_probe(m, 6, P.fp16(), None, 5000, 1)
    done.append("step-error probe")
    L.density_histogram(lin, 1, 200000, lin.max_value(), 0.05, 200)
    L.density_histogram(None, 1, 50000, 8.0, 0.05, 20000)  # global-memory bins
    done.append("density (shared and global bins)")
    runs = [(l, P.fp16() if l % 2 else P.fp32(), bool(l % 3 == 0), 500 + 700 * l, l << 40)
            for l in range(6)]
    L.run_coupled_many(m, lin, 2, runs)
    done.append("multi-run")
    print("sanitize ok:", "; ".join(done))


if __name__ == "__main__":
    main()
