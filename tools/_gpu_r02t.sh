timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shard.py -q -rfE -s > gpurun_out/r02t_pytest.log 2>&1
python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02t_c4.log 2>&1
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02t_c3.log 2>&1
timeout 600 python bench.py > gpurun_out/r02t_bench.jsonl 2>gpurun_out/r02t_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02t_bench_ref.jsonl 2>gpurun_out/r02t_bench_ref.err
