cd $GRAFT_REPO_ROOT
O=gpurun_out/r02ab2; mkdir -p $O
for lib in "" paper_2012_09739_b200/liblpmc_b200_grp2.so paper_2012_09739_b200/liblpmc_b200_midfirst.so; do
echo "lib=$lib" >> $O/timing.log
t() { echo "$1 $(LPMC_LIB=$lib timeout 300 python tools/profile_level.py --time "${@:2}" 2>&1 | tail -1)" >> $O/timing.log; }
t c4-l12-fp16 --level 12 --prec fp16 --payoff call --n 4194304 --base $((12<<40))
t c4-l12-fp32 --level 12 --prec fp32 --payoff call --n 4194304 --base $((12<<40 | 2<<36))
t c4-l11-fp32 --level 11 --prec fp32 --payoff call --n 4194304 --base $((11<<40 | 2<<36))
t c4-l4-fp32 --level 4 --prec fp32 --payoff call --n 16777216 --base $((4<<40 | 2<<36))
done
cat $O/timing.log
