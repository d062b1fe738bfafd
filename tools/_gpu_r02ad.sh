cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_shard.py tests/test_gpu_parity.py -x -q -rfE > gpurun_out/r02ad_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r02ad_tests.log
timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -rfE > gpurun_out/r02ad_configs.log 2>&1; echo configs rc=$?; tail -2 gpurun_out/r02ad_configs.log
echo "== C4 A/B" > gpurun_out/r02ad_ab.txt
bash tools/ab_time.sh --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 >> gpurun_out/r02ad_ab.txt 2>&1
echo "== C4 new static" >> gpurun_out/r02ad_ab.txt
KNN_B200_TRI_DYN=0 timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 >> gpurun_out/r02ad_ab.txt 2>&1
echo "== C2 A/B" >> gpurun_out/r02ad_ab.txt
bash tools/ab_time.sh --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/r02ad_ab.txt 2>&1
echo "== C2 new static" >> gpurun_out/r02ad_ab.txt
KNN_B200_TRI_DYN=0 timeout 300 python tools/profile_solve.py --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/r02ad_ab.txt 2>&1
echo "== C3 A/B" >> gpurun_out/r02ad_ab.txt
bash tools/ab_time.sh --n 1000000 --d 1024 --k 100 --seed 2 --reps 2 >> gpurun_out/r02ad_ab.txt 2>&1
for m in 0 2 3 4; do
KNN_B200_DEBUG_SWEEP_ONLY=1 KNN_B200_DEBUG_SWEEP=$m timeout 600 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 1 --reps 1 > gpurun_out/r02ad_c4_mode$m.jsonl 2>&1; echo c4 mode $m rc=$?
KNN_B200_DEBUG_SWEEP_ONLY=1 KNN_B200_DEBUG_SWEEP=$m timeout 600 python tools/shard_emulate.py --worlds 1 --reps 1 > gpurun_out/r02ad_c2_mode$m.jsonl 2>&1; echo c2 mode $m rc=$?
done
