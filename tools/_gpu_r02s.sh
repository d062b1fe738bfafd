timeout 2000 python -m pytest tests -m gpu -q -rfE --durations=15 > gpurun_out/r02s_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1
python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02s_c3.log 2>&1
python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02s_c4.log 2>&1
