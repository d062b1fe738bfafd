timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -rfE -k "threshold" > gpurun_out/r02v_pytest.log 2>&1
timeout 900 python -m pytest tests/test_gpu_configs.py -q -rfE -s -k "c3 or c4 or clusters or near_ties or equal" >> gpurun_out/r02v_pytest.log 2>&1
python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02v_c4.log 2>&1
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02v_c3.log 2>&1
