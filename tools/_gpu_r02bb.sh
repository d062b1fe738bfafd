cd $GRAFT_REPO_ROOT
TAG=r02bb
M=gpu__time_duration.sum,sm__cycles_active.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tc.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:tensor_sweep_kernel --launch-skip 2 -c 2 --csv python tools/profile_solve.py --n 1000000 --reps 2 > gpurun_out/${TAG}_c2_pipe.csv 2>&1; echo ncu rc=$?
for c in "--n 1000000" "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
  echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
done
timeout 1500 python -m pytest tests -m gpu -q -rfE -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; cut -c1-250 gpurun_out/${TAG}_bench_c2.jsonl
