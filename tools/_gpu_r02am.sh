cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_configs.py -x -q -rfE -k "not c5 and not past_2_32" > gpurun_out/r02am_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r02am_tests.log
echo "== C2" > gpurun_out/r02am_ab.txt
bash tools/ab_multi.sh "base new" --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/r02am_ab.txt 2>&1
KNN_B200_TRI_DYN=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 -o gpurun_out/r02am_tri_c2_dyn python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/r02am_ncu.log 2>&1; echo ncu rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02am_c2_launches.csv python tools/profile_solve.py --n 1000000 --reps 1 > /dev/null 2>&1; echo ncu2 rc=$?
