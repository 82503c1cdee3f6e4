"""Per-kernel table of the ncu demand files (tools/ncu_capture.sh output or
profiles/r02_*_demands.json) for DESIGN.md / profiles summaries.

    python tools/ncu_table.py peaks.json file.json [file.json ...]

peaks.json: {"fp64_ops_per_s": ..., "fp32_ops_per_s": ..., "fp16_ops_per_s": ...}
(bench.py's pipe_peaks_measured).  Rates use the ncu launch duration.
"""
from __future__ import annotations

import json
import sys


def main():
    peaks = json.load(open(sys.argv[1]))
    print("| kernel (launch) | ms (ncu) | path-steps/s | warp-inst / warp-step | FP64 lane-ops / "
          "path-step | FP64 % of peak | issue active % | FP64 pipe % | FMA pipe inst % | "
          "ALU pipe inst % | smem wavefronts / path-step | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for f in sys.argv[2:]:
        d = json.load(open(f))
        ps = d["path_steps_per_launch"]
        rate = ps / (d["ncu_duration_ms"] * 1e-3)
        fp64 = d["fp64_lane_ops_per_path_step"] * rate / peaks["fp64_ops_per_s"]
        c = d["co_limits"]
        name = f.split("/")[-1].replace("_demands.json", "").replace(".json", "")
        print(f"| {name} | {d['ncu_duration_ms']:.2f} | {rate:.3e} | "
              f"{32 * d['warp_inst_per_path_step']:.1f} | {d['fp64_lane_ops_per_path_step']:.2f} | "
              f"{100 * fp64:.1f} | {c['issue_active_pct']:.1f} | {c['fp64_pipe_active_pct']:.1f} | "
              f"{c['fma_pipe_inst_pct']:.1f} | {c['alu_pipe_inst_pct']:.1f} | "
              f"{d['smem_wavefronts_per_path_step']:.2f} | {d['registers_per_thread']:.0f} |")


if __name__ == "__main__":
    main()
