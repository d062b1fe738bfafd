cd $GRAFT_REPO_ROOT
for lib in base new; do
  if [ $lib = new ]; then unset KNN_B200_LIB; else export KNN_B200_LIB=$PWD/paper_0906_0231_b200/lib/libknn_b200_$lib.so; fi
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:tensor_sweep_kernel --launch-skip 1 -c 1 -o gpurun_out/r02ag_c2tri_$lib python tools/profile_solve.py --n 1000000 --reps 1 > gpurun_out/r02ag_ncu_$lib.log 2>&1; echo ncu $lib rc=$?
done
