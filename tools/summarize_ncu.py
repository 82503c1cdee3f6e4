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
]


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
    else:
        print(full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None))
