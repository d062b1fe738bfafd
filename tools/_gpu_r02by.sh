# packed FADD2/FMUL2 fold terms: GPU suite on the new build, then old-vs-new timings
cd $GRAFT_REPO_ROOT
TAG=r02by
timeout 2000 python -m pytest tests -m gpu -q -rfE -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${TAG}_pytest_gpu.log
cp paper_0906_0231_b200/lib/libknn_b200.so /tmp/new.so
run() { echo "$1 | $2" >> gpurun_out/${TAG}_ab.txt; timeout 300 python tools/profile_solve.py $2 --reps 3 >> gpurun_out/${TAG}_ab.txt 2>&1; }
for v in old new old new; do
  if [ $v = old ]; then cp alt_lib/libknn_b200_old.so paper_0906_0231_b200/lib/libknn_b200.so; else cp /tmp/new.so paper_0906_0231_b200/lib/libknn_b200.so; fi
  run $v "--n 131072 --d 256 --k 10 --arith exact --seed 1"
  run $v "--n 65536 --d 128 --k 32 --metric cosine --arith exact --seed 3"
  run $v "--n 1000000 --d 256 --k 10 --seed 1"
  run $v "--n 1000000 --d 1024 --k 100 --seed 2"
  run $v "--n 4000000 --d 128 --k 32 --metric cosine --seed 3"
done
cp /tmp/new.so paper_0906_0231_b200/lib/libknn_b200.so
