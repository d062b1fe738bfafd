cd $GRAFT_REPO_ROOT
TAG=r02al
timeout 2400 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference_c2.jsonl 2> gpurun_out/${TAG}_ref.err; echo ref rc=$?
for c in "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
  echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_l.log 2>&1; echo ncu launches rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 -o gpurun_out/${TAG}_tri_c2 python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo ncu full rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 -o gpurun_out/${TAG}_tri_c4 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 > gpurun_out/${TAG}_ncu_full4.log 2>&1; echo ncu full4 rc=$?
