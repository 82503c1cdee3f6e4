"""Time the C2 sweep through the public API two ways: a per-level loop of
run_coupled_paths vs one run_coupled_many call (diagnostic)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_09739_b200 as L

model = L.make_gbm(); spec = L.PrecisionSpec.fp32(); approx = L.InvCdfApprox.parse("linear:16")
n = 1 << 22
cfgs = [(l, k) for l in range(11) for k in (False, True)]
runs = [(l, spec, k, n, (l << 40) | (int(k) << 39)) for (l, k) in cfgs]
def loop():
    for (l, spec_, k, nn, b) in runs:
        L.run_coupled_paths(model, l, spec_, approx, k, nn, 1, b, device=0)
def many():
    L.run_coupled_many(model, approx, 1, runs, device=0)
def many_sorted():  # biggest first
    L.run_coupled_many(model, approx, 1, sorted(runs, key=lambda r: -r[0]), device=0)
for f in (loop, many, many_sorted, loop, many):
    f()
    t = time.perf_counter(); f(); f(); dt = (time.perf_counter() - t) / 2
    print(f"{f.__name__:12s} {dt*1e3:8.2f} ms  {n * sum(1 << l for l, _ in cfgs) / dt:.4e} path-steps/s", flush=True)
