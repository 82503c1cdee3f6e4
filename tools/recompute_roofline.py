"""Recompute a bench line's `roofline` block from its own achieved value and
the per-path-step demands in profiles/fp64_ops_per_path_step.json (used when
the ncu capture that sets those demands ran in the same GPU call as the bench,
i.e. after the bench had read the previous constants).  Same formulas as
bench.py.

    python tools/recompute_roofline.py gpurun_out/bench_v18.json > profiles/r01_bench_v18.json
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_SM = 148


def main() -> None:
    line = [l for l in open(sys.argv[1]) if l.startswith("{")][-1]
    out = json.loads(line)
    prof = json.load(open(os.path.join(ROOT, "profiles", "fp64_ops_per_path_step.json")))
    roof = out["roofline"]
    achieved = roof["achieved"]
    sm_hz = (out.get("clocks", {}).get("sm_mhz") or 1965.0) * 1e6
    peaks = {"fp64": out["pipe_peaks_measured"]["fp64_ops_per_s"], "issue": 4.0 * N_SM * sm_hz,
             "smem": 1.0 * N_SM * sm_hz}
    demand = {"fp64": prof["fp64_lane_ops_per_path_step"],
              "issue": prof["warp_inst_per_path_step"],
              "smem": prof["smem_wavefronts_per_path_step"]}
    for k, p in roof["pipes"].items():
        p["demand_per_path_step"] = demand[k]
        p["peak_per_s"] = peaks[k]
        p["ceiling_path_steps_per_s"] = peaks[k] / demand[k]
        p["frac"] = achieved / p["ceiling_path_steps_per_s"]
    bind = min(roof["pipes"], key=lambda k: roof["pipes"][k]["ceiling_path_steps_per_s"])
    roof["bound"] = f"multi-pipe non-tensor (binding: {bind})"
    roof["peak"] = roof["pipes"][bind]["ceiling_path_steps_per_s"]
    roof["frac"] = achieved / roof["peak"]
    roof["fp64_frac"] = roof["pipes"]["fp64"]["frac"]
    roof["traffic"] = prof.get("dram_bytes_per_launch")
    roof["co_limits"] = prof.get("co_limits")
    roof["recomputed"] = (f"pipes/peak/frac/traffic/co_limits recomputed from the run's own "
                          f"achieved value with the demands of {prof.get('source')} "
                          f"(tools/recompute_roofline.py)")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
