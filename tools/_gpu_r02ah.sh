cd $GRAFT_REPO_ROOT
echo "== C2" > gpurun_out/r02ah_ab.txt
bash tools/ab_multi.sh "base new nodyn noudone" --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/r02ah_ab.txt 2>&1
echo "== C2 new static" >> gpurun_out/r02ah_ab.txt
KNN_B200_TRI_DYN=0 timeout 300 python tools/profile_solve.py --n 1000000 --d 256 --k 10 --seed 1 --reps 3 >> gpurun_out/r02ah_ab.txt 2>&1
for lib in new nodyn; do
  if [ $lib = new ]; then unset KNN_B200_LIB; else export KNN_B200_LIB=$PWD/paper_0906_0231_b200/lib/libknn_b200_$lib.so; fi
  timeout 600 ncu --section SpeedOfLight --section WarpStateStats --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg,dram__bytes_read.sum --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/r02ah_ncu_$lib.txt 2>&1; echo ncu $lib rc=$?
done
