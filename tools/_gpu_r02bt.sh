cd $GRAFT_REPO_ROOT
TAG=r02bt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_shard.py -m gpu -q -rfE -k "threshold or c3 or c4 or capture or rescore or cluster or outlier or near_ties or equal_norms" > gpurun_out/${TAG}_pytest_band.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_band.log
C3="--n 1000000 --d 1024 --k 100 --seed 2"; C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
for c in "$C3" "$C4" "$C3" "$C4"; do echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__registers_per_thread,launch__grid_size,launch__block_size
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore_capture" --csv python tools/profile_solve.py $C3 --reps 1 > gpurun_out/${TAG}_c3_rescore.csv 2>&1; echo c3 ncu rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore_capture" --csv python tools/profile_solve.py $C4 --reps 1 > gpurun_out/${TAG}_c4_rescore.csv 2>&1; echo c4 ncu rc=$?
