cd $GRAFT_REPO_ROOT
TAG=r02ba
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum
for mode in 2 5 7; do
  KNN_B200_DEBUG_SWEEP=$mode KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py --n 1000000 --reps 2 > gpurun_out/${TAG}_mode$mode.csv 2>&1; echo mode $mode rc=$?
done
