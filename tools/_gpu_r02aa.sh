cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r02aa_bench.jsonl 2>gpurun_out/r02aa_bench.err; echo bench rc=$?
timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 > gpurun_out/r02aa_c4.log 2>&1; echo c4 rc=$?
rm -f gpurun_out/r02aa_cta_w8.txt gpurun_out/r02aa_cta_w1.txt
KNN_B200_DEBUG_CTA_TIMES=gpurun_out/r02aa_cta_w8.txt timeout 900 python tools/shard_emulate.py --worlds 8 --reps 0 > gpurun_out/r02aa_shard.jsonl 2>&1; echo sh8 rc=$?
KNN_B200_DEBUG_CTA_TIMES=gpurun_out/r02aa_cta_w1.txt timeout 900 python tools/shard_emulate.py --worlds 1 --reps 0 >> gpurun_out/r02aa_shard.jsonl 2>&1; echo sh1 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 -o gpurun_out/r02aa_c4tri python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 1 > gpurun_out/r02aa_ncu_c4.log 2>&1; echo ncu rc=$?
