"""Benchmark of the B200 MLMC level-correction sampler (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--scaling weak|strong]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Workload (BASELINE.json configs[3], "C4" -- the largest single-GPU config):
nested-MLMC four-way difference P_f,exact - P_c,exact - P_f,approx + P_c,approx
for GBM dS = 0.05 S dt + 0.2 S dW, S0 = 1, T = 1, European call payoff
max(S_T - 1, 0); exact Gaussians in fp64 (hat legs) and approximate ones
(linear:16 table) in the reference's fp16 (m = 10 semantics, run on native binary16) and fp32 (bar
legs); levels 0..12; 2^24 paths per level per GPU (weak scaling; --scaling
strong keeps 2^24 paths per level in total; --paths changes either).  Every path runs all four
coupled legs and all three moment families (estimate_level_stats semantics,
mlmc.hpp:113-149).  Precisions and path bases follow the reference's
four-way experiment (experiments.hpp:170-213): low = fp16 at l << 40, high =
fp32 at l << 40 | 2 << 36.  One "step" = 13 levels x 2 precisions = 26 level
launches (2.75e11 fine path-steps per GPU).

metric: fine path-steps per second (paths x 2^level, summed over the sweep).
value:  device-timed (CUDA events on the launching stream), parameters and
        tables already resident, max over ranks.
e2e:    through the public multi-run API (lpmc_run_coupled_many_partials on
        this rank's chunk range of every run, the same call for every N) +
        all_gather + index-order fold + LevelStats per run, host buffers,
        wall clock with syncs, max over ranks.
C2 (BASELINE configs[1]) is measured too and reported under "c2".
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Euler-Maruyama path-steps/sec per MLMC level & precision; % of FP roofline"
UNIT = "path-steps/s"
LEVELS = list(range(0, 13))
PRECS = ("fp16", "fp32")  # the four-way experiment's low / high roles
PATHS_PER_GPU = 1 << 24
SEED = 1
STRIKE = 1.0
APPROX = "linear:16"
WORKLOAD = ("BASELINE config 4: nested-MLMC 4-way difference, GBM(mu=0.05, sigma=0.2, S0=1, T=1), "
            "European call payoff max(S_T-1,0), exact fp64 Gaussians + linear:16 approximate "
            "Gaussians in fp16 (the reference's m=10 semantics) and fp32, no Kahan, levels 0..12, "
            "2^24 paths per level, all four coupled legs -> d_hat, d_bar, d_four moments")
DEMANDS = os.path.join(ROOT, "profiles", "r02_c4_l12_demands.json")
CPU_SAMPLE = 1 << 15  # >= 256 paths x threads x 8 at 16 threads

C2_LEVELS = list(range(0, 11))
C2_PATHS = 1 << 22


def path_base(level: int, prec: str) -> int:
    return (level << 40) | ((2 << 36) if prec == "fp32" else 0)


def mbits(prec: str) -> int:
    return 10 if prec == "fp16" else 23


def fine_steps(level: int, n: int) -> int:
    return n << level


def host_info() -> dict:
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count(),
            "glibc": " ".join(platform.libc_ver())}


# --------------------------------------------------------------- clocks -----
class ClockSampler:
    """nvidia-smi sampling during the timed region (recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx.append(float(parts[2]))
                except ValueError:
                    continue
                for name, v in zip(names, parts[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ reference -----
def _cpu_runner():
    """The reference's own CPU run_coupled_paths (oracle/_ref, the unmodified
    /root/reference headers compiled by oracle/Makefile); the oracle port if
    _ref is absent.  The reference has no payoff option: it runs the terminal
    payoff, a free post-step on the same four legs (mlmc.hpp:86-90)."""
    from oracle.bind import Oracle, Reference
    threads = os.cpu_count() or 1
    if Reference.available():
        R = Reference()

        def one(level, prec, n):
            rc, msg, _ = R.run_coupled_paths(level=level, mantissa_bits=mbits(prec), approx=APPROX,
                                             kahan=False, n=n, seed=SEED,
                                             path_base=path_base(level, prec), threads=threads)
            assert rc == 0, msg
        return one, "reference", threads
    O = Oracle()

    def one(level, prec, n):
        cfg = O.config(level=level, mantissa_bits=mbits(prec), approx=APPROX, kahan=False,
                       seed=SEED)
        rc, _, _ = O.run_sequential(cfg, n, path_base(level, prec), threads=threads)
        assert rc == 0
    return one, "port", threads


def run_reference(args, rank: int) -> None:
    """--impl reference: the reference's CPU path on all host cores, on a
    bounded sample of the same workload: step i runs precision PRECS[i % 2]
    over levels 0..12 at 2^15 paths per level (both precisions alternate, so
    any two consecutive steps cover the C4 mix)."""
    if rank != 0:
        return
    one, kind, threads = _cpu_runner()

    def step(i):
        prec = PRECS[i % 2]
        for l in LEVELS:
            one(l, prec, CPU_SAMPLE)
        return sum(fine_steps(l, CPU_SAMPLE) for l in LEVELS)

    for i in range(args.warmup):
        step(i)
    work = 0
    t0 = time.perf_counter()
    for i in range(args.steps):
        work += step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = work / dt
    desc = (f"{CPU_SAMPLE} paths per (level 0..12, precision); step i runs one precision "
            f"(fp16, fp32 alternating), all four legs, terminal payoff (the reference has no call "
            f"payoff: a free post-step); {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64+f32+f16(m=10)",
            "data": "synthetic (seeded counter RNG)", "impl": "reference",
            "config": {"workload": WORKLOAD, "sample_paths_per_level": CPU_SAMPLE},
            "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                                  "sample": desc}, **host_info()),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample() -> dict:
    """The reference timed on this host on a bounded sample (~10-30 s)."""
    one, kind, threads = _cpu_runner()
    work = sum(fine_steps(l, CPU_SAMPLE) for l in LEVELS) * len(PRECS)
    t0 = time.perf_counter()
    for prec in PRECS:
        for l in LEVELS:
            one(l, prec, CPU_SAMPLE)
    dt = time.perf_counter() - t0
    return dict({"value": work / dt, "unit": UNIT, "cores": threads, "kind": kind,
                 "sample": f"{CPU_SAMPLE} paths per (level 0..12, fp16/fp32) = {work:.3e} fine "
                           f"path-steps, all four legs, terminal payoff, {dt:.2f} s wall on "
                           f"{threads} threads"}, **host_info())


# ------------------------------------------------------------- roofline -----
# FP64 operations per fine path-step of the reference's
# algorithm (FMA-free source-level count): RNG 2 + exact Z ~130 + approximate
# Z 5 + carrier legs 11.5.
ALGORITHMIC_FP64_PER_PATH_STEP = 148.5


def roofline(L, per_cfg_ms, cfgs, n_local, clk, peaks, n_sm):
    """Roofline of the dominant kernel (no HBM or tensor bound: state lives in
    registers).  frac = executed FP64 lane-ops/s (ncu-counted per fine
    path-step x live path-steps/s) / measured FP64 peak -- the north-star
    figure, which falls when FP64 work is removed.  algorithmic = the
    contract's definition (SURVEY 8(d)'s per-unit figure x units / time).
    dispatch = the resource that binds the kernel: the SM sub-partition's
    issue/dispatch port, where an FP64 warp-instruction occupies two slots
    (profiles/r02_dispatch_model.md)."""
    from paper_2012_09739_b200.build import kernel_source_hash
    dom = max(cfgs, key=lambda c: statistics.mean(per_cfg_ms[c]))
    dom_ms = statistics.mean(per_cfg_ms[dom])
    rate = fine_steps(dom[0], n_local) / (dom_ms * 1e-3)  # path-steps/s, CUDA events
    prof = {}
    if os.path.exists(DEMANDS):
        with open(DEMANDS) as f:
            prof = json.load(f)
    src_hash = kernel_source_hash()
    stale = prof.get("kernel_source_hash") != src_hash
    sm_hz = (clk.get("sm_mhz") or 1965.0) * 1e6
    pipes = {}
    if prof.get("fp64_lane_ops_per_path_step"):
        pipes["fp64"] = {"demand_per_path_step": prof["fp64_lane_ops_per_path_step"],
                         "peak_per_s": peaks["fp64_ops_per_s"], "unit": "FP64 lane-ops"}
    if prof.get("warp_inst_per_path_step"):
        pipes["issue"] = {"demand_per_path_step": prof["warp_inst_per_path_step"],
                          "peak_per_s": 4.0 * n_sm * sm_hz, "unit": "warp-instructions"}
    if prof.get("warp_inst_per_path_step") and prof.get("fp64_warp_inst_per_path_step"):
        pipes["dispatch"] = {"demand_per_path_step": prof["warp_inst_per_path_step"] +
                             prof["fp64_warp_inst_per_path_step"],
                             "peak_per_s": 4.0 * n_sm * sm_hz,
                             "unit": "dispatch slots (an FP64 warp-instruction takes two)"}
    if prof.get("smem_wavefronts_per_path_step"):
        pipes["smem"] = {"demand_per_path_step": prof["smem_wavefronts_per_path_step"],
                         "peak_per_s": 1.0 * n_sm * sm_hz, "unit": "shared-memory wavefronts"}
    for p in pipes.values():
        p["ceiling_path_steps_per_s"] = p["peak_per_s"] / p["demand_per_path_step"]
        p["frac"] = rate / p["ceiling_path_steps_per_s"]
    kernel = f"level_kernel level {dom[0]} {dom[1]} (all legs, call payoff, linear:16)"
    alg = ALGORITHMIC_FP64_PER_PATH_STEP * rate
    algorithmic = {"fp64_ops_per_path_step": ALGORITHMIC_FP64_PER_PATH_STEP,
                   "achieved": alg / 1e12, "frac": alg / peaks["fp64_ops_per_s"],
                   "note": "SURVEY.md 8(d) count of the reference's algorithm (Acklam + Newton on "
                           "libm erfc/exp ~130 FP64 per Gaussian); > 1 because the device "
                           "computes the same Gaussians from a direct table in 10"}
    if "fp64" not in pipes:
        return {"bound": "fp64", "achieved": None, "peak": peaks["fp64_ops_per_s"] / 1e12,
                "unit": "TFLOP/s", "frac": None, "traffic": None, "kernel": kernel,
                "path_steps_per_s": rate, "algorithmic": algorithmic,
                "note": "per-path-step demands not profiled"}
    achieved = pipes["fp64"]["demand_per_path_step"] * rate  # FP64 lane-ops/s
    bind = min(pipes, key=lambda k: pipes[k]["ceiling_path_steps_per_s"])
    return {
        "bound": "fp64", "achieved": achieved / 1e12, "peak": peaks["fp64_ops_per_s"] / 1e12,
        "unit": "TFLOP/s", "frac": achieved / peaks["fp64_ops_per_s"],
        "traffic": prof.get("dram_bytes_per_launch"), "kernel": kernel,
        "path_steps_per_s": rate, "launch_ms": dom_ms,
        "fp64_lane_ops_per_path_step": pipes["fp64"]["demand_per_path_step"],
        "demands": os.path.relpath(DEMANDS, ROOT), "demands_stale": stale,
        "kernel_source_hash": src_hash,
        "algorithmic": algorithmic,
        # an FP64 warp-instruction holds the sub-partition's dispatch port for two cycles:
        # with this instruction mix the FP64 fraction cannot exceed 2 N64 / (N + N64)
        "fp64_frac_at_full_dispatch": 2.0 * prof["fp64_warp_inst_per_path_step"] /
        pipes["dispatch"]["demand_per_path_step"] if "dispatch" in pipes else None,
        "dispatch_frac": pipes["dispatch"]["frac"] if "dispatch" in pipes else None,
        "multi_pipe": {"binding": bind, "frac": pipes[bind]["frac"],
                       "ceiling_path_steps_per_s": pipes[bind]["ceiling_path_steps_per_s"],
                       "pipes": pipes, "co_limits": prof.get("co_limits")},
        "note": "no HBM or tensor bound: per-path state lives in registers (traffic = DRAM bytes "
                "of one launch, ncu). achieved = executed FP64 lane-ops per fine path-step (ncu "
                "sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}, one lane-op per DFMA as the "
                "pipe issues it) x the dominant launch's path-steps/s from CUDA events; peak = "
                "FP64 lane-op rate measured live on this GPU (lpmc_measure_pipe_peaks; "
                "MEASURED_PEAKS.json has no FP64 figure), in 1e12 lane-ops/s. frac falls when "
                "FP64 work is removed (round 2 cut the exact Gaussian from 40 to 10 FP64 "
                "operations and the kernel got 1.5x faster); algorithmic uses SURVEY 8(d)'s "
                "count instead. dispatch_frac = used / available dispatch slots, an FP64 "
                "warp-instruction counted twice: the resource that binds this kernel. "
                "demands_stale = the profiled kernel sources differ from this build."}


# ------------------------------------------------------------------ ours ----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--paths", type=int, default=PATHS_PER_GPU,
                    help="paths per level: per GPU (weak) or in total (strong); a multiple of "
                         "2^18 (e.g. 2^30 for the C5 strong-scaling total)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist

    import paper_2012_09739_b200 as L
    from paper_2012_09739_b200.sharded import allgather_partials, shard_chunks

    # LPMC_BENCH_SHARED_GPU=1: functional test of the multi-rank flow on a
    # one-GPU box (every rank on cuda:0, gloo collectives on host tensors).
    # Its numbers are not a scaling measurement and are never reported.
    shared = os.environ.get("LPMC_BENCH_SHARED_GPU") == "1"
    gpu_index = 0 if shared else local
    torch.cuda.set_device(gpu_index)
    dev = torch.device("cuda", gpu_index)
    coll_dev = None if shared else dev
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    model = L.make_gbm(0.05, 0.2, 1.0, 1.0)
    specs = {"fp16": L.PrecisionSpec.fp16(), "fp32": L.PrecisionSpec.fp32()}
    approx = L.InvCdfApprox.parse(APPROX)
    if args.paths % (1 << 18):
        raise SystemExit("--paths must be a multiple of 2^18 (one chunk)")
    n_total = args.paths * (world if args.scaling == "weak" else 1)
    n_chunks = n_total // (1 << 18)
    c0, c1 = shard_chunks(n_chunks, rank, world)
    n_local = (c1 - c0) * (1 << 18)
    cfgs = [(l, p) for l in LEVELS for p in PRECS]
    ext = dict(payoff="call", strike=STRIKE)
    plans = {(l, p): L.LevelPlan(model, l, specs[p], approx, False, n_total, SEED, path_base(l, p),
                                 chunks=(c0, c1), device=gpu_index, **ext) for (l, p) in cfgs}
    # A dedicated stream: torch's legacy default stream has handle 0, which
    # the C-ABI reads as "the plan's own stream".
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    sptr = stream.cuda_stream
    assert sptr != 0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def sweep(pl, keys, events=None):
        for c in keys:
            if events is not None:
                events[c][0].record(stream)
            pl[c].launch(sptr)
            if events is not None:
                events[c][1].record(stream)

    def gather_all(pl, keys, nck):
        out = {}
        for c in keys:
            part = pl[c].collect_partials()
            full = allgather_partials(part, nck, None, coll_dev) if world > 1 else part
            out[c] = L.fold_partials(full)
        return out

    def timed(pl, keys, steps, nck):
        per_step, per_cfg = [], {c: [] for c in keys}
        res = None
        barrier()
        torch.cuda.synchronize(dev)
        for _ in range(steps):
            flush.zero_()  # L2 flush (256 MiB > 126 MB L2), outside the events
            ev = {c: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for c in keys}
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            sweep(pl, keys, ev)
            t1.record(stream)
            torch.cuda.synchronize(dev)
            per_step.append(t0.elapsed_time(t1))
            for c in keys:
                per_cfg[c].append(ev[c][0].elapsed_time(ev[c][1]))
            res = gather_all(pl, keys, nck)  # results of every timed step are produced
        barrier()
        torch.cuda.synchronize(dev)
        return per_step, per_cfg, res

    # warm-up (also a correctness pass of the collective path)
    for _ in range(max(args.warmup, 1)):
        sweep(plans, cfgs)
        torch.cuda.synchronize(dev)
        results = gather_all(plans, cfgs, n_chunks)

    clocks = ClockSampler(gpu_index)
    if rank == 0:
        clocks.start()
    L.reset_launch_count()
    per_step_ms, per_cfg_ms, results = timed(plans, cfgs, args.steps, n_chunks)
    launches = L.launch_count()
    clk = clocks.stop() if rank == 0 else {}

    def max_over_ranks(x: float) -> float:
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    step_ms_max = max_over_ranks(sum(per_step_ms) / len(per_step_ms))
    work_total = sum(fine_steps(l, n_total) for (l, p) in cfgs)
    value = work_total / (step_ms_max * 1e-3)

    # ---- e2e through the public multi-run API (the same call for every N) ----
    e2e_steps = max(1, min(args.steps, 3))
    runs = [(l, specs[p], False, n_total, path_base(l, p)) for (l, p) in cfgs]
    ranges = [(c0, c1)] * len(runs)

    def e2e_step():
        parts = L.run_coupled_many_partials(model, approx, SEED, runs, ranges,
                                            device=gpu_index, **ext)
        for (l, p), part in zip(cfgs, parts):
            full = allgather_partials(part, n_chunks, None, coll_dev) if world > 1 else part
            L.level_stats_from_moments(L.fold_partials(full), l, specs[p], False, n_total)

    e2e_step()  # untimed warm-up: stream pool, pinned staging and buffers are created once
    torch.cuda.synchronize(dev)
    barrier()
    w0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize(dev)
    barrier()
    e2e_value = work_total / max_over_ranks((time.perf_counter() - w0) / e2e_steps)
    table_bytes = 7 * 16 * 8  # linear:16 breakpoints, coefficients and scalars
    h2d = len(cfgs) * (table_bytes + 12)  # table + failure-word/flag init per run
    d2h = len(cfgs) * ((c1 - c0) * 15 * 8 + 12)  # chunk partials + failure word/flag per run

    # ---- C2 (BASELINE configs[1]) as a secondary line ------------------------
    c2 = None
    if not args.no_c2:
        c2_total = C2_PATHS * (world if args.scaling == "weak" else 1)
        c2_chunks = c2_total // (1 << 18)
        d0, d1 = shard_chunks(c2_chunks, rank, world)
        c2_cfgs = [(l, k) for l in C2_LEVELS for k in (False, True)]
        fp32 = specs["fp32"]
        c2_plans = {(l, k): L.LevelPlan(model, l, fp32, approx, k, c2_total, SEED,
                                        (l << 40) | (int(k) << 36), chunks=(d0, d1),
                                        device=gpu_index) for (l, k) in c2_cfgs}
        sweep(c2_plans, c2_cfgs)
        torch.cuda.synchronize(dev)
        gather_all(c2_plans, c2_cfgs, c2_chunks)
        c2_steps, _, _ = timed(c2_plans, c2_cfgs, max(3, min(args.steps, 10)), c2_chunks)
        c2_ms = max_over_ranks(statistics.mean(c2_steps))
        c2 = {"workload": "BASELINE config 2: levels 0..10, fp32 linear:16, +-Kahan, 2^22 paths per "
                          "level per GPU, terminal payoff, all four legs",
              "value": sum(fine_steps(l, c2_total) for (l, k) in c2_cfgs) / (c2_ms * 1e-3),
              "unit": UNIT, "ms_per_step": c2_ms}
        for p in c2_plans.values():
            p.close()

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = L.measure_pipe_peaks(gpu_index)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    roof = roofline(L, per_cfg_ms, cfgs, n_local, clk, peaks, n_sm)
    cpu = None if args.no_cpu_baseline else cpu_baseline_sample()
    per_level = {p: {} for p in PRECS}
    for (l, p) in cfgs:
        per_level[p][str(l)] = fine_steps(l, n_local) / (statistics.mean(per_cfg_ms[(l, p)]) * 1e-3)
    top = results[(12, "fp16")], results[(12, "fp32")]
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
           "scaling": args.scaling, "vs_baseline": None, "dtype": "f64+f32+f16(m=10)",
           "data": "synthetic (seeded counter-based RNG; no dataset)",
           "config": {"workload": WORKLOAD,
                      "paths_per_level": n_total, "paths_per_level_per_gpu": n_local,
                      "levels": "0..12", "precisions": ["fp16 (the reference's m=10 semantics, on native binary16 with static scales)", "fp32"],
                      "kahan": False, "approx": APPROX, "payoff": "call, strike 1",
                      "legs": "all", "reduce": "tree",
                      "path_bases": "fp16: l<<40, fp32: l<<40 | 2<<36 (experiments.hpp:185-194)",
                      "parallelism": f"paths sharded by 2^18-path chunks over {world} GPU(s); "
                                     "one all_gather of chunk moments per run",
                      "l2": "flushed between timed steps (256 MiB write); kernels read no "
                            "input tensors"},
           "gpu_launches": int(launches),
           "clocks": clk,
           "roofline": roof,
           "pipe_peaks_measured": peaks,
           "per_level_path_steps_per_s_per_gpu": per_level,
           "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": d2h,
                   "method": "lpmc_run_coupled_many_partials over the rank's chunk range of all "
                             "26 runs (concurrent on the device's stream pool), all_gather, fold, "
                             "LevelStats; wall clock, max over ranks"},
           "cpu_baseline": cpu,
           "c2": c2,
           "check": {"v_hat_l12": top[0].d_hat.variance(),
                     "v_bar_l12_fp16": top[0].d_bar.variance(),
                     "V_bar_l12_fp16": top[0].d_four.variance(),
                     "V_bar_l12_fp32": top[1].d_four.variance()}}
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
