cd $GRAFT_REPO_ROOT
TAG=r02bf
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2"
KNN_B200_DEBUG_SWEEP=4 KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py $C4 > gpurun_out/${TAG}_c4_mode4.csv 2>&1; echo rc=$?
KNN_B200_DEBUG_SWEEP=2 KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py $C4 > gpurun_out/${TAG}_c4_mode2.csv 2>&1; echo rc=$?
KNN_B200_TCAP_EW=16 KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py $C4 > gpurun_out/${TAG}_c4_ew16.csv 2>&1; echo rc=$?
echo "ew8" > gpurun_out/${TAG}_c4_time.txt; timeout 300 python tools/profile_solve.py $C4 >> gpurun_out/${TAG}_c4_time.txt 2>&1
echo "ew16" >> gpurun_out/${TAG}_c4_time.txt; KNN_B200_TCAP_EW=16 timeout 300 python tools/profile_solve.py $C4 >> gpurun_out/${TAG}_c4_time.txt 2>&1
