cd $GRAFT_REPO_ROOT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build/tmem_bw tools/tmem_bw.cu && timeout 120 ./build/tmem_bw > gpurun_out/r02ab_tmem_bw.txt 2>&1; echo tmem rc=$?
for m in 0 1 2 4; do
KNN_B200_DEBUG_SWEEP_ONLY=1 KNN_B200_DEBUG_SWEEP=$m timeout 600 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 1 --reps 1 > gpurun_out/r02ab_c4_mode$m.jsonl 2>&1; echo mode $m rc=$?
done
KNN_B200_DEBUG_SWEEP_ONLY=1 timeout 600 python tools/shard_emulate.py --n 1000000 --d 1024 --k 100 --seed 2 --worlds 1 --reps 1 > gpurun_out/r02ab_c3_mode0.jsonl 2>&1; echo c3 rc=$?
