cd $GRAFT_REPO_ROOT
TAG=r02bv
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_configs.py -m gpu -q -rfE -x > gpurun_out/${TAG}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest.log
C2="--n 1000000 --d 256 --k 10 --seed 1"
for v in 1 0 1 0; do echo "COOP=$v" >> gpurun_out/${TAG}_c2.txt; KNN_B200_RESCORE_COOP=$v timeout 300 python tools/profile_solve.py $C2 --reps 4 >> gpurun_out/${TAG}_c2.txt 2>&1; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers,launch__registers_per_thread,launch__grid_size
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore_kernel" --csv python tools/profile_solve.py $C2 --reps 1 > gpurun_out/${TAG}_c2_rescore.csv 2>&1; echo ncu rc=$?
