cd $GRAFT_REPO_ROOT
TAG=r02br
cp paper_0906_0231_b200/lib/libknn_b200.so /tmp/s3.so
for s in 3 4 3 4; do
  cp /tmp/s3.so paper_0906_0231_b200/lib/libknn_b200.so; [ $s = 4 ] && cp alt_lib/libknn_b200_s4.so paper_0906_0231_b200/lib/libknn_b200.so
  for c in "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
    echo "S=$s $c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__registers_per_thread,launch__grid_size,launch__block_size
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore_capture" --csv python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > gpurun_out/${TAG}_c3_rescore_s4.csv 2>&1; echo c3 ncu rc=$?
cp /tmp/s3.so paper_0906_0231_b200/lib/libknn_b200.so
