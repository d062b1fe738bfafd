cd $GRAFT_REPO_ROOT
TAG=r02bk
timeout 1500 python tools/shard_emulate.py --n 16000000 --d 256 --k 10 --seed 4 --worlds 8 --reps 1 > gpurun_out/${TAG}_shard_c5.jsonl 2>&1; echo emu5 rc=$?; tail -1 gpurun_out/${TAG}_shard_c5.jsonl | cut -c1-300
