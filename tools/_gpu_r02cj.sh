# list triangle at one GPU: static walk (default) vs the unit queue
cd $GRAFT_REPO_ROOT
TAG=r02cj
C2="--n 1000000 --d 256 --k 10 --seed 1"
run() { echo "$1 | $2" >> gpurun_out/${TAG}_knobs.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 4 >> gpurun_out/${TAG}_knobs.txt 2>&1; }
for r in 1 2; do run "X=default" "$C2"; run "KNN_B200_TRI_DYN=1" "$C2"; done
