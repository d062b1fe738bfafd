cd $GRAFT_REPO_ROOT
TAG=r02at
summ() { python -c 'import json,sys
for l in sys.stdin:
    if not l.startswith("{"): continue
    d=json.loads(l)
    if "world" in d: print(d["world"], d["bit_identical_to_single_gpu"], round(d["max_rank_ms"],2), d["est_speedup"], [[round(x,2) for x in p] for p in d["rank_ms_phases[prep,sample,sweep+bin,merge]"]])
    else: print(d["T1_ms"])'; }
for kv in "X=0" "KNN_B200_TRI_TAIL=10" "KNN_B200_TRI_TAIL=30" "KNN_B200_TRI_DYN=0" "X=0" "KNN_B200_TRI_TAIL=30"; do
  echo "$kv" >> gpurun_out/${TAG}_w8.txt
  env $kv timeout 600 python tools/shard_emulate.py --worlds 4,8 --reps 2 2>&1 | summ >> gpurun_out/${TAG}_w8.txt
done
KNN_B200_DEBUG_CTA_TIMES=gpurun_out/${TAG}_cta_head.txt timeout 600 python tools/shard_emulate.py --worlds 8 --reps 0 > /dev/null 2>&1; echo cta rc=$?
echo "world1 head" >> gpurun_out/${TAG}_w8.txt
KNN_B200_TRI_WALK=2 timeout 600 python tools/shard_emulate.py --worlds 1 --reps 2 2>&1 | summ >> gpurun_out/${TAG}_w8.txt
timeout 900 python -m pytest tests/test_gpu_shard.py -q -rfE -x > gpurun_out/${TAG}_pytest_shard.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_shard.log
