"""Diagnostic: level-10 wall time per call with and without torch's CUDA
context created first, and over repeated calls (clock ramp)."""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if "--torch" in sys.argv:
    import torch
    torch.cuda.init(); torch.zeros(1, device="cuda")
import paper_2012_09739_b200 as L
model = L.make_gbm(); spec = L.PrecisionSpec.fp32(); approx = L.InvCdfApprox.parse("linear:16")
n = 1 << 22
plan = L.LevelPlan(model, 10, spec, approx, False, n, 1, 0)
for i in range(12):
    t = time.perf_counter(); plan.launch(); plan.collect(); dt = time.perf_counter() - t
    if i % 3 == 0:
        clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    else:
        clk = ""
    print(f"{'torch' if '--torch' in sys.argv else 'plain'} call {i:2d} {dt*1e3:8.3f} ms {clk}", flush=True)
