# last knob sweep: threshold-triangle sample rank (C3, C4), hub weight (C2)
cd $GRAFT_REPO_ROOT
TAG=r02ci
C2="--n 1000000 --d 256 --k 10 --seed 1"; C3="--n 1000000 --d 1024 --k 100 --seed 2"; C4="--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
run() { echo "$1 | $2" >> gpurun_out/${TAG}_knobs.txt; env $1 timeout 300 python tools/profile_solve.py $2 --reps 3 >> gpurun_out/${TAG}_knobs.txt 2>&1; }
run "X=default" "$C4"; run "KNN_B200_TCAP_RANK=6" "$C4"; run "KNN_B200_TCAP_RANK=8" "$C4"
run "X=default" "$C3"; run "KNN_B200_TCAP_RANK=8" "$C3"; run "KNN_B200_TCAP_RANK=10" "$C3"
run "X=default" "$C2"; run "KNN_B200_TRI_HUB=0" "$C2"; run "KNN_B200_TRI_HUB=150" "$C2"; run "X=default" "$C2"
