timeout 900 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 1,2,4,8 --reps 1 > gpurun_out/r02u_shard_emulate_c4.jsonl 2>&1
timeout 900 python tools/shard_emulate.py --n 1000000 --d 1024 --k 100 --seed 2 --worlds 1,8 --reps 1 > gpurun_out/r02u_shard_emulate_c3.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02u_c2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02u_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tensor_sweep --launch-skip 1 --launch-count 1 -o gpurun_out/r02u_c2_tri python tools/profile_solve.py --n 1000000 --d 256 --k 10 --seed 1 --reps 1 > gpurun_out/r02u_ncu_full.log 2>&1
