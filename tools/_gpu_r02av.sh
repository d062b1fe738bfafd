cd $GRAFT_REPO_ROOT
TAG=r02av
timeout 1500 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; cut -c1-250 gpurun_out/${TAG}_bench_c2.jsonl
timeout 900 python tools/shard_emulate.py --worlds 1,2,4,8 --reps 3 > gpurun_out/${TAG}_shard_c2.jsonl 2>&1; echo emu rc=$?
timeout 900 python tools/shard_emulate.py --n 1000000 --d 1024 --k 100 --seed 2 --worlds 8 --reps 2 > gpurun_out/${TAG}_shard_c3.jsonl 2>&1; echo emu3 rc=$?
timeout 900 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 2,4,8 --reps 2 > gpurun_out/${TAG}_shard_c4.jsonl 2>&1; echo emu4 rc=$?
for c in "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
  echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
done
