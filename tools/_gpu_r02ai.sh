cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_configs.py -x -q -rfE -k "not c5 and not past_2_32" > gpurun_out/r02ai_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r02ai_tests.log
echo "== C2" > gpurun_out/r02ai_ab.txt
bash tools/ab_multi.sh "base new" --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/r02ai_ab.txt 2>&1
echo "== C4" >> gpurun_out/r02ai_ab.txt
bash tools/ab_multi.sh "base new" --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 >> gpurun_out/r02ai_ab.txt 2>&1
echo "== C3" >> gpurun_out/r02ai_ab.txt
bash tools/ab_multi.sh "base new" --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 >> gpurun_out/r02ai_ab.txt 2>&1
timeout 600 python tools/shard_emulate.py --worlds 1,8 --reps 2 > gpurun_out/r02ai_shard_c2.jsonl 2>&1; echo emu rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:rescore_capture --launch-skip 0 -c 1 -o gpurun_out/r02ai_c3_band python tools/profile_solve.py --n 1000000 --d 1024 --k 100 --seed 2 --reps 1 > gpurun_out/r02ai_ncu_c3.log 2>&1; echo ncu rc=$?
