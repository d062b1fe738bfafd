# C2 rescore: rank-based phase-1 selection vs k + 4 warp-minimum rounds
cd $GRAFT_REPO_ROOT
TAG=r02cb
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -q -rfE -x > gpurun_out/${TAG}_pytest.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest.log
cp paper_0906_0231_b200/lib/libknn_b200.so /tmp/new.so
M=gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread
for v in old new old new; do
  if [ $v = old ]; then cp alt_lib/libknn_b200_old.so paper_0906_0231_b200/lib/libknn_b200.so; else cp /tmp/new.so paper_0906_0231_b200/lib/libknn_b200.so; fi
  echo "$v" >> gpurun_out/${TAG}_ab.txt; timeout 300 python tools/profile_solve.py --n 1000000 --reps 4 >> gpurun_out/${TAG}_ab.txt 2>&1
  timeout 600 ncu --metrics $M --clock-control none -k regex:"rescore_kernel" --csv python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/${TAG}_${v}_rescore.csv 2>&1
  grep -h "gpu__time_duration" gpurun_out/${TAG}_${v}_rescore.csv >> gpurun_out/${TAG}_ab.txt
done
cp /tmp/new.so paper_0906_0231_b200/lib/libknn_b200.so
