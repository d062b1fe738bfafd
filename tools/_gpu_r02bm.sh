cd $GRAFT_REPO_ROOT
TAG=r02bm
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__registers_per_thread,launch__grid_size,launch__block_size,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore" --csv python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/${TAG}_c2_rescore.csv 2>&1; echo c2 rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore" --csv python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > gpurun_out/${TAG}_c3_rescore.csv 2>&1; echo c3 rc=$?
