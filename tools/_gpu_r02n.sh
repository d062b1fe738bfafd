set -x
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -rfE -k "triangle or loopback or nccl or multi or c2 or threshold or golden or random or long" > gpurun_out/r02n_pytest.log 2>&1
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02n_c3.log 2>&1
python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02n_c4.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02n_bench.jsonl 2>gpurun_out/r02n_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tensor_sweep --launch-skip 1 --launch-count 1 -o gpurun_out/r02n_c4_tcap python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 > gpurun_out/r02n_ncu.log 2>&1
