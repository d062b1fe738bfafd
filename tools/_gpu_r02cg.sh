# streamed threshold triangle (C3): unit queue x column-group size; C2/C4 group size
cd $GRAFT_REPO_ROOT
TAG=r02cg
C2="--n 1000000 --d 256 --k 10 --seed 1"; C3="--n 1000000 --d 1024 --k 100 --seed 2"; C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
run() { echo "$1 | $2" >> gpurun_out/${TAG}_knobs.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 3 >> gpurun_out/${TAG}_knobs.txt 2>&1; }
run "X=default" "$C3"
for g in 10 20 30 40; do run "KNN_B200_TRI_DYN=1 KNN_B200_TRI_GROUP_MB=$g" "$C3"; done
run "KNN_B200_TRI_DYN=0 KNN_B200_TRI_GROUP_MB=20" "$C3"
run "X=default" "$C3"
for g in 20 30 40; do run "KNN_B200_TRI_GROUP_MB=$g" "$C4"; done
for g in 20 30 40; do run "KNN_B200_TRI_GROUP_MB=$g" "$C2"; done
