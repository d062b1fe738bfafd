cd $GRAFT_REPO_ROOT
TAG=r02bu
C2="--n 1000000 --d 256 --k 10 --seed 1"
run() { echo "$1 | $2" >> gpurun_out/${TAG}_c2knobs.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 4 >> gpurun_out/${TAG}_c2knobs.txt 2>&1; }
for r in 1 2; do
run "X=default" "$C2"
run "KNN_B200_TRI_STRIDE=32 KNN_B200_TRI_RANK=2" "$C2"
run "KNN_B200_TRI_STRIDE=32 KNN_B200_TRI_RANK=3" "$C2"
run "KNN_B200_TRI_STRIDE=8 KNN_B200_TRI_RANK=4" "$C2"
run "KNN_B200_KPL=14" "$C2"
run "KNN_B200_TRI_RANK=3" "$C2"
done
