# ncu co-limit counters of the C2 level-10 launch for several nvcc define
# variants (VARIANTS="default -DX ..."): shared-memory wavefronts and bank
# conflicts, issue activity, FP64 pipe, stall reasons per issue.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/ncu_variants_${1:-x}.csv
: > $OUT
M=gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio
for V in ${VARIANTS}; do
  [ "$V" = "default" ] && V=""
  LPMC_NVCC_EXTRA="$(echo $V | tr ',' ' ')" python -m paper_2012_09739_b200.build --force > gpurun_out/build_variant.log 2>&1 || { echo "BUILD FAILED $V" >> $OUT; continue; }
  timeout 300 python tools/profile_level.py > /dev/null 2>&1 || { echo "RUN FAILED $V" >> $OUT; continue; }
  echo "# variant [$V]" >> $OUT
  timeout 900 ncu --clock-control none --metrics $M -k regex:level_kernel -s 1 -c 1 --csv python tools/profile_level.py 2>/dev/null | grep -v "^==" | grep '"' >> $OUT
done
python - "$OUT" <<'EOF'
import csv, sys
rows, var = [], None
for line in open(sys.argv[1]):
    if line.startswith("#"):
        var = line.strip()[2:]
        continue
    r = next(csv.reader([line]))
    if len(r) > 3 and r[0] != "ID":
        rows.append((var, r[-3], r[-1]))
for v, m, x in rows:
    print(v, m, x)
EOF
