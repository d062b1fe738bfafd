cd $GRAFT_REPO_ROOT
TAG=r02ap
C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3 --reps 2"
for kv in "X=0" "KNN_B200_TCAP_RANK=6" "KNN_B200_TCAP_RANK=8" "KNN_B200_TCAP_RANK=9" "KNN_B200_TCAP_STRIDE=24" "KNN_B200_TCAP_STRIDE=32" "KNN_B200_TCAP_STRIDE=32 KNN_B200_TCAP_RANK=5" "KNN_B200_TCAP_STRIDE=12" "KNN_B200_TCAP_CAP=512" "X=0"; do
  echo "$kv $(env $kv timeout -s KILL 300 python tools/profile_solve.py $C4 2>&1 | tail -1 | cut -c1-160)" >> gpurun_out/${TAG}_c4_knobs.txt
done
