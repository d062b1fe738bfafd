timeout 2400 python -m pytest tests -m gpu -q -rfE -x > gpurun_out/r02y_pytest_gpu.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02y_bench.jsonl 2>gpurun_out/r02y_bench.err
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02y_c3.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02y_c2_launches.csv python tools/profile_solve.py --n 1000000 --d 256 --k 10 --seed 1 --reps 1 > /dev/null 2>&1
timeout 900 python tools/shard_emulate.py --worlds 8 --reps 2 > gpurun_out/r02y_shard_c2.jsonl 2>&1
