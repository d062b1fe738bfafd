rm -f gpurun_out/r02z_cta_w8.txt gpurun_out/r02z_cta_w1.txt
KNN_B200_DEBUG_CTA_TIMES=gpurun_out/r02z_cta_w8.txt timeout 900 python tools/shard_emulate.py --worlds 8 --reps 0 > gpurun_out/r02z_shard.jsonl 2>&1
KNN_B200_DEBUG_CTA_TIMES=gpurun_out/r02z_cta_w1.txt timeout 900 python tools/shard_emulate.py --worlds 1 --reps 0 >> gpurun_out/r02z_shard.jsonl 2>&1
