"""Fixed per-call overhead of the public API (diagnostic): wall time per call
of run_coupled_paths / level_partials / a prebuilt LevelPlan on a level-0 run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2012_09739_b200 as L

model = L.make_gbm(); spec = L.PrecisionSpec.fp32(); approx = L.InvCdfApprox.parse("linear:16")
for n in (1 << 10, 1 << 22):
    for lvl in (0, 10):
        if lvl == 10 and n < 1 << 20: continue
        plan = L.LevelPlan(model, lvl, spec, approx, False, n, 1, 0)
        fs = {"run_coupled_paths": lambda: L.run_coupled_paths(model, lvl, spec, approx, False, n, 1, 0, device=0),
              "level_partials": lambda: L.level_partials(model, lvl, spec, approx, False, n, 1, 0, 0, (n + 262143) // 262144, device=0),
              "plan launch+collect": lambda: (plan.launch(), plan.collect())}
        for name, f in fs.items():
            f(); f()
            reps = 20 if lvl == 0 else 3
            t = time.perf_counter()
            for _ in range(reps): f()
            dt = (time.perf_counter() - t) / reps
            print(f"n={n:8d} level={lvl:2d} {name:20s} {dt*1e3:8.3f} ms/call", flush=True)
        plan.close()
