cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_configs.py -x -q -rfE -k "c4 or loopback or forced or pool or gaussian" > gpurun_out/r02an_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r02an_tests.log
echo "== C2 dyn forced" > gpurun_out/r02an_ab.txt
KNN_B200_TRI_DYN=1 bash tools/ab_multi.sh "prev new" --n 1000000 --d 256 --k 10 --seed 1 --reps 2 >> gpurun_out/r02an_ab.txt 2>&1
echo "== C2 default" >> gpurun_out/r02an_ab.txt
bash tools/ab_multi.sh "new" --n 1000000 --d 256 --k 10 --seed 1 --reps 2 >> gpurun_out/r02an_ab.txt 2>&1
echo "== C4" >> gpurun_out/r02an_ab.txt
bash tools/ab_multi.sh "prev new" --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 >> gpurun_out/r02an_ab.txt 2>&1
timeout 600 python tools/shard_emulate.py --worlds 1,8 --reps 2 > gpurun_out/r02an_shard_c2.jsonl 2>&1; echo emu rc=$?
