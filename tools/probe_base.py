"""Diagnostic: level-10 launch time vs path_base / seed / stream (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2012_09739_b200 as L
model = L.make_gbm(); spec = L.PrecisionSpec.fp32(); approx = L.InvCdfApprox.parse("linear:16")
n = 1 << 22
st = torch.cuda.Stream()
for seed, base in ((1, 0), (1, 10 << 40), (2, 0), (1, 12345), (7, 10 << 40), (1, 0)):
    plan = L.LevelPlan(model, 10, spec, approx, False, n, seed, base)
    res = []
    for _ in range(4):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); plan.launch(st.cuda_stream); e1.record(st); torch.cuda.synchronize(); plan.collect()
        res.append(e0.elapsed_time(e1))
    plan.close()
    print(f"seed={seed} base={base:#x} ms={' '.join(f'{x:.3f}' for x in res)}", flush=True)
