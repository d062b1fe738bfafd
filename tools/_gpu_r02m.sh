set -x
timeout 600 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -q -rfE -x -k "triangle or loopback or nccl or multi or c2 or threshold or golden or random" > gpurun_out/r02m_pytest.log 2>&1
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02m_c3.log 2>&1
python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02m_c4.log 2>&1
KNN_B200_TCAP_CAP=1024 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02m_c4_cap1024.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02m_c3_launches.csv python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > /dev/null 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02m_bench.jsonl 2>gpurun_out/r02m_bench.err
