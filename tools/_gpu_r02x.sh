timeout 1500 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -rfE -s > gpurun_out/r02x_pytest.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02x_bench.jsonl 2>gpurun_out/r02x_bench.err
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02x_c3.log 2>&1
python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02x_c4.log 2>&1
