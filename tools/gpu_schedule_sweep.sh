# fused vs warp-per-path time per level launch (the auto schedule's crossover)
cd $GRAFT_REPO_ROOT
for cfg in "12 1250" "11 2500" "10 5000" "9 10000" "8 10000" "6 10000" "4 10000" "3 10000" "10 20000" "10 40000" "6 40000"; do
  set -- $cfg
  for sch in fused warp_per_path; do
    echo "level $1 n $2 $sch two-way-fp16-l1024 $(python tools/profile_level.py --time --level $1 --n $2 --prec fp16 --approx linear:1024 --legs fine --schedule $sch | tail -1) | all-fp32-l16 $(python tools/profile_level.py --time --level $1 --n $2 --schedule $sch | tail -1)"
  done
done
