cd $GRAFT_REPO_ROOT
TAG=r02bs
C3="--n 1000000 --d 1024 --k 100 --seed 2"; C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
cp paper_0906_0231_b200/lib/libknn_b200.so /tmp/def.so
run() { echo "$1 | $2" >> gpurun_out/${TAG}_configs.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1; }
for s in def s2 def s2; do
  cp /tmp/def.so paper_0906_0231_b200/lib/libknn_b200.so; [ $s = s2 ] && cp alt_lib/libknn_b200_s2.so paper_0906_0231_b200/lib/libknn_b200.so
  run "LIB=$s" "$C3"; run "LIB=$s" "$C4"
done
cp /tmp/def.so paper_0906_0231_b200/lib/libknn_b200.so
run "KNN_B200_TCAP_STRIDE=32" "$C4"; run "KNN_B200_TCAP_STRIDE=8" "$C4"; run "KNN_B200_TCAP_STRIDE=64" "$C3"; run "KNN_B200_TCAP_STRIDE=16" "$C3"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__occupancy_limit_shared_mem,launch__registers_per_thread,launch__grid_size,launch__block_size
timeout 900 ncu --metrics $M --clock-control none -k regex:"rescore_capture" --csv python tools/profile_solve.py $C3 --reps 1 > gpurun_out/${TAG}_c3_rescore.csv 2>&1; echo c3 ncu rc=$?
