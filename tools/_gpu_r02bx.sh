cd $GRAFT_REPO_ROOT
TAG=r02bx
KNN_B200_DEBUG_FB=1 timeout 900 python tools/shard_emulate.py --n 1000000 --d 1024 --k 100 --seed 2 --worlds 8 --reps 1 > gpurun_out/${TAG}_shard_c3.jsonl 2> gpurun_out/${TAG}_c3_fb.txt; echo emu3 rc=$?
KNN_B200_DEBUG_FB=1 timeout 900 python tools/shard_emulate.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --worlds 8 --reps 1 > gpurun_out/${TAG}_shard_c4.jsonl 2> gpurun_out/${TAG}_c4_fb.txt; echo emu4 rc=$?
