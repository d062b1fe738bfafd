# threshold triangle knob sweep on the last build: column-group size, walk
cd $GRAFT_REPO_ROOT
TAG=r02cf
C3="--n 1000000 --d 1024 --k 100 --seed 2"; C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
run() { echo "$1 | $2" >> gpurun_out/${TAG}_knobs.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 3 >> gpurun_out/${TAG}_knobs.txt 2>&1; }
for c in "$C4" "$C3"; do
  run "X=default" "$c"
  run "KNN_B200_TRI_GROUP_MB=20" "$c"
  run "KNN_B200_TRI_GROUP_MB=80" "$c"
  run "KNN_B200_TRI_DYN=0" "$c"
  run "KNN_B200_TRI_DYN=1" "$c"
  run "X=default" "$c"
done
