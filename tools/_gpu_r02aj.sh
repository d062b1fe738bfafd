cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_shard.py tests/test_gpu_parity.py -x -q -rfE -k "not c5 and not past_2_32" > gpurun_out/r02aj_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r02aj_tests.log
echo "== C4" > gpurun_out/r02aj_ab.txt
bash tools/ab_multi.sh "base new" --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 >> gpurun_out/r02aj_ab.txt 2>&1
echo "== C3" >> gpurun_out/r02aj_ab.txt
bash tools/ab_multi.sh "base new" --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 >> gpurun_out/r02aj_ab.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02aj_c3_launches.csv python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > /dev/null 2>&1; echo ncu3 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02aj_c4_launches.csv python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 > /dev/null 2>&1; echo ncu4 rc=$?
