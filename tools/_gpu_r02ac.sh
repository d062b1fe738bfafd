cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_shard.py -x -q -rfE > gpurun_out/r02ac_shard_tests.log 2>&1; echo shard tests rc=$?; tail -2 gpurun_out/r02ac_shard_tests.log
timeout 1200 python -m pytest tests/test_gpu_configs.py -x -q -rfE -k "c3 or c4 or gaussian or outlier or equal_norms" > gpurun_out/r02ac_configs.log 2>&1; echo configs rc=$?; tail -2 gpurun_out/r02ac_configs.log
timeout 600 python tools/shard_emulate.py --worlds 1,8 --reps 2 > gpurun_out/r02ac_shard_c2_dyn.jsonl 2>&1; echo emu dyn rc=$?
KNN_B200_TRI_DYN=0 timeout 600 python tools/shard_emulate.py --worlds 8 --reps 2 > gpurun_out/r02ac_shard_c2_static.jsonl 2>&1; echo emu static rc=$?
timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02ac_c4_dyn.log 2>&1; echo c4 rc=$?
KNN_B200_TRI_DYN=0 timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02ac_c4_static.log 2>&1; echo c4s rc=$?
KNN_B200_TCAP_STRIDE=32 timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02ac_c4_s32.log 2>&1; echo c4 s32 rc=$?
timeout 300 python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 > gpurun_out/r02ac_c3_dyn.log 2>&1; echo c3 rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02ac_c4_launches.csv python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 > /dev/null 2>&1; echo ncu rc=$?
