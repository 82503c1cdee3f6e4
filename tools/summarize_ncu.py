"""Summaries of ncu output for profiles/ (run here, on the CPU box).

    python tools/summarize_ncu.py launches gpurun_out/launches.csv
    python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep [path_steps]
"""
from __future__ import annotations

import collections
import csv
import io
import re
import subprocess
import sys


def kernel_key(name: str) -> str:
    m = re.search(r"level_kernel<([^>]*)>", name)
    if m:
        return "level_kernel<" + m.group(1).replace("lpmc_b200::<unnamed>::", "") + ">"
    return name.split("(")[0].replace("void ", "").split("::")[-1]


def launches(path: str) -> str:
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = {k: i for i, k in enumerate(rows[0])}
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[h["Metric Name"]] != "gpu__time_duration.sum":
            continue
        us = float(r[h["Metric Value"]].replace(",", "")) * scale.get(r[h["Metric Unit"]], 1.0)
        k = kernel_key(r[h["Kernel Name"]])
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {n} | {us / 1e3:.3f} | {us / tot:.2%} |")
    return "\n".join(out)


WANT = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp16_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_hadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_hmul_pred_on.sum",
    "sm__sass_thread_inst_executed_op_hfma_pred_on.sum",
    "sm__sass_thread_inst_executed_op_integer_pred_on.sum",
    "launch__occupancy_limit_shared_mem", "launch__shared_mem_per_block_static",
]


def raw_values(path: str) -> tuple[str, dict, dict]:
    """(kernel name, metric -> float, metric -> unit) of the first kernel."""
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, v = rows[0], rows[1], rows[2]
    vals, us = {}, {}
    for i, name in enumerate(h):
        try:
            vals[name] = float(v[i].replace(",", ""))
            us[name] = units[i]
        except ValueError:
            pass
    return v[h.index("Kernel Name")], vals, us


def demands(path: str, path_steps: float, note: str) -> str:
    """Per-fine-path-step demands of one profiled launch, the JSON bench.py
    reads (profiles/r02_c4_l12_demands.json); tied to the kernel sources by
    their hash."""
    import json
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2012_09739_b200.build import kernel_source_hash
    name, v, u = raw_values(path)
    fp64 = sum(v.get(f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum", 0.0)
               for o in ("dadd", "dmul", "dfma"))
    dur = v["gpu__time_duration.sum"] * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
                                         "nsecond": 1e-6, "ms": 1.0, "msecond": 1.0}.get(
        u["gpu__time_duration.sum"], 1.0)
    out = {
        "kernel": kernel_key(name), "note": note, "path_steps_per_launch": path_steps,
        "ncu_duration_ms": dur,
        "fp64_lane_ops_per_path_step": round(fp64 / path_steps, 3),
        "warp_inst_per_path_step": round(v["smsp__inst_executed.sum"] / path_steps, 4),
        "fp64_warp_inst_per_path_step": round(
            v.get("sm__inst_executed_pipe_fp64.sum", 0.0) / path_steps, 4),
        "smem_wavefronts_per_path_step": round(
            v.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0) / path_steps, 4),
        "dram_bytes_per_launch": v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0),
        "registers_per_thread": v.get("launch__registers_per_thread"),
        "co_limits": {
            "issue_active_pct": v.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_active_pct": v.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "smem_wavefronts_pct_of_peak": v.get(
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "fma_pipe_inst_pct": v.get("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
            "alu_pipe_inst_pct": v.get("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "xu_pipe_pct": v.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
            "bank_conflicts": v.get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        },
        "definition": "ncu --set full of one launch: FP64 lane-ops = sm__sass_thread_inst_executed_"
                      "op_{dadd,dmul,dfma}_pred_on.sum, warp-instructions = smsp__inst_executed.sum (FP64 pipe: "
                      "sm__inst_executed_pipe_fp64.sum), "
                      "shared-memory wavefronts = l1tex__data_pipe_lsu_wavefronts_mem_shared.sum, "
                      "each / fine path-steps of the launch; DRAM = dram__bytes_read.sum + "
                      "dram__bytes_write.sum",
        "kernel_source_hash": kernel_source_hash(),
    }
    return json.dumps(out, indent=1)


def full(path: str, path_steps: float | None) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        kname = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"### `{kernel_key(kname)}`\n")
        out.append("| metric | unit | value |\n|---|---|---|")
        vals = {}
        for name in WANT:
            if name in h:
                i = h.index(name)
                out.append(f"| {name} | {units[i]} | {v[i]} |")
                try:
                    vals[name] = float(v[i].replace(",", ""))
                except ValueError:
                    pass
        if path_steps:
            fp64 = sum(vals.get(f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum", 0.0)
                       for o in ("dadd", "dmul", "dfma"))
            warp = vals.get("smsp__inst_executed.sum", 0.0)
            warp64 = vals.get("sm__inst_executed_pipe_fp64.sum", 0.0)
            out.append(f"| derived: fp64 lane-ops per path-step | | {fp64 / path_steps:.2f} |")
            out.append(f"| derived: warp-instructions per warp-step | | "
                       f"{warp / (path_steps / 32):.1f} |")
            out.append(f"| derived: fp64 warp-instructions per warp-step | | "
                       f"{warp64 / (path_steps / 32):.1f} |")
        out.append("")
        # opcode mix from the source page
        src = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                              "sass"], capture_output=True, text=True).stdout
        srows = list(csv.reader(io.StringIO(src)))
        hdr = [i for i, r in enumerate(srows[:8]) if "Address" in r and "Source" in r]
        if hdr and path_steps:
            srows = srows[hdr[0]:]
            sh = srows[0]
            iS, iE = sh.index("Source"), sh.index("Instructions Executed")
            iW = sh.index("Warp Stall Sampling (All Samples)")
            by, st = collections.Counter(), collections.Counter()
            for r in srows[1:]:
                if len(r) <= iE:
                    continue
                try:
                    n = int(r[iE])
                except ValueError:
                    continue
                s = re.sub(r"^@!?U?P\w+\s+", "", r[iS].strip())
                op = s.split()[0].split(".")[0] if s else "?"
                by[op] += n
                st[op] += int(r[iW] or 0)
            out.append("| opcode | warp-inst per warp-step | stall samples |\n|---|---|---|")
            for k, n in by.most_common(25):
                out.append(f"| {k} | {n / (path_steps / 32):.2f} | {st[k]} |")
            out.append("")
        break
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    elif sys.argv[1] == "demands":
        print(demands(sys.argv[2], float(sys.argv[3]), sys.argv[4] if len(sys.argv) > 4 else ""))
    else:
        print(full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None))
