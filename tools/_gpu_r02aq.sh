cd $GRAFT_REPO_ROOT
TAG=r02aq
timeout 1500 python -m pytest tests -m gpu -q -rfE -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python tools/shard_emulate.py --worlds 1,8 --reps 2 > gpurun_out/${TAG}_shard_c2.jsonl 2>&1; echo emu rc=$?
KNN_B200_TRI_DYN=0 timeout 600 python tools/shard_emulate.py --worlds 8 --reps 2 > gpurun_out/${TAG}_shard_c2_static.jsonl 2>&1; echo emu2 rc=$?
KNN_B200_DEBUG_CTA_TIMES=gpurun_out/${TAG}_cta_dyn.txt timeout 600 python tools/shard_emulate.py --worlds 8 --reps 0 > /dev/null 2>&1; echo cta rc=$?
KNN_B200_TRI_DYN=0 KNN_B200_DEBUG_CTA_TIMES=gpurun_out/${TAG}_cta_static.txt timeout 600 python tools/shard_emulate.py --worlds 8 --reps 0 > /dev/null 2>&1; echo cta2 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_c2_launches.csv python tools/profile_solve.py --n 1000000 --reps 2 > /dev/null 2>&1; echo ncu rc=$?
