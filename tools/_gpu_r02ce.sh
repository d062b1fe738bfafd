# 16 epilogue warps by default in the threshold triangle: GPU suite, C3/C4 steps
cd $GRAFT_REPO_ROOT
TAG=r02ce
timeout 2000 python -m pytest tests -m gpu -q -rfE > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo smoke rc=$?
for c in "--n 1000000 --d 1024 --k 100 --seed 2" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"; do
  echo "$c" >> gpurun_out/${TAG}_configs.txt; timeout 300 python tools/profile_solve.py $c --reps 3 >> gpurun_out/${TAG}_configs.txt 2>&1
done
timeout 900 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 8 --reps 1 > gpurun_out/${TAG}_shard_c4.jsonl 2>&1; echo emu4 rc=$?
