# threshold triangle: 8 vs 16 epilogue warps at C3 and C4
cd $GRAFT_REPO_ROOT
TAG=r02cd
run() { echo "$1 | $2" >> gpurun_out/${TAG}_ew.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 3 >> gpurun_out/${TAG}_ew.txt 2>&1; }
for r in 1 2; do
for ew in 8 16; do
  run "KNN_B200_TCAP_EW=$ew" "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
  run "KNN_B200_TCAP_EW=$ew" "--n 1000000 --d 1024 --k 100 --seed 2"
done; done
