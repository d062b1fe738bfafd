# unit queue for the streamed threshold triangle too: GPU suite, smoke, C3/C4 steps, C3 sharded emulation, bench
cd $GRAFT_REPO_ROOT
TAG=r02ch
timeout 2000 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
for c in "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
  echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
done
timeout 900 python tools/shard_emulate.py --n 1000000 --d 1024 --k 100 --seed 2 --worlds 8 --reps 2 > gpurun_out/${TAG}_shard_c3.jsonl 2>&1; echo emu3 rc=$?
timeout 600 python bench.py > gpurun_out/${TAG}_bench_c2.jsonl 2> gpurun_out/${TAG}_bench.err; echo bench rc=$?; cut -c1-200 gpurun_out/${TAG}_bench_c2.jsonl
