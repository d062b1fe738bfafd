cd $GRAFT_REPO_ROOT
TAG=r02bc
timeout 900 python tools/shard_emulate.py --worlds 1,2,4,8 --reps 3 > gpurun_out/${TAG}_shard_c2.jsonl 2>&1; echo emu rc=$?
timeout 900 python tools/shard_emulate.py --n 1000000 --d 1024 --k 100 --seed 2 --worlds 8 --reps 2 > gpurun_out/${TAG}_shard_c3.jsonl 2>&1; echo emu3 rc=$?
timeout 900 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 2,4,8 --reps 2 > gpurun_out/${TAG}_shard_c4.jsonl 2>&1; echo emu4 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/${TAG}_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_l.log 2>&1; echo ncu launches rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 -o gpurun_out/${TAG}_tri_c2 python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo ncu full rc=$?
