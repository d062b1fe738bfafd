cd $GRAFT_REPO_ROOT
KNN_B200_TCAP_EW=16 timeout 900 python -m pytest tests/test_gpu_configs.py -x -q -rfE -k "c4 or gaussian or outlier or equal_norms" > gpurun_out/r02ak_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r02ak_tests.log
for rep in 1 2; do
echo "ew8 $(timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 | tail -1 | cut -c1-70)" >> gpurun_out/r02ak_ab.txt
echo "ew16 $(KNN_B200_TCAP_EW=16 timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 | tail -1 | cut -c1-70)" >> gpurun_out/r02ak_ab.txt
done
for m in 0 2 4; do
KNN_B200_TCAP_EW=16 KNN_B200_DEBUG_SWEEP_ONLY=1 KNN_B200_DEBUG_SWEEP=$m timeout 600 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 1 --reps 1 > gpurun_out/r02ak_c4_ew16_mode$m.jsonl 2>&1; echo c4 mode $m rc=$?
done
