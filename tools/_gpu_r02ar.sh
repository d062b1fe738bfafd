cd $GRAFT_REPO_ROOT
TAG=r02ar
for g in 10 20 40 80; do
  echo "G=$g $(KNN_B200_TRI_GROUP_MB=$g timeout 600 python tools/shard_emulate.py --worlds 8 --reps 2 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["max_rank_ms"], d["est_speedup"], [round(p[2],1) for p in d["rank_ms_phases[prep,sample,sweep+bin,merge]"]])')" >> gpurun_out/${TAG}_group_w8.txt
done
for g in 20 40 80 20 40 80; do
  echo "G=$g $(KNN_B200_TRI_GROUP_MB=$g timeout 300 python tools/profile_solve.py --n 1000000 --reps 2 2>&1 | tail -1 | cut -c1-100)" >> gpurun_out/${TAG}_group_c2.txt
done
for g in 20 40 20 40; do
  echo "G=$g $(KNN_B200_TRI_GROUP_MB=$g timeout 300 python tools/profile_solve.py --n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2 2>&1 | tail -1 | cut -c1-100)" >> gpurun_out/${TAG}_group_c4.txt
done
