cd $GRAFT_REPO_ROOT
TAG=r02bd
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
for mode in 0 2 3 4; do
  KNN_B200_DEBUG_SWEEP=$mode KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py --n 1000000 --reps 2 > gpurun_out/${TAG}_mode$mode.csv 2>&1; echo mode $mode rc=$?
done
for mode in 0 3; do
  KNN_B200_DEBUG_SWEEP=$mode KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/${TAG}_c4_mode$mode.csv 2>&1; echo c4 mode $mode rc=$?
done
