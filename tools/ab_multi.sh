#!/bin/bash
# Same-box timing of several in-tree library builds (dev tool):
#   ab_multi.sh "base new nodyn ..." [profile_solve args]   (lib/libknn_b200_<name>.so; "new" = libknn_b200.so)
cd "$(dirname "$0")/.."
libs=$1; shift
for rep in 1 2; do
for lib in $libs; do
  if [ $lib = new ]; then unset KNN_B200_LIB; else export KNN_B200_LIB=$PWD/paper_0906_0231_b200/lib/libknn_b200_$lib.so; fi
  echo "$lib $(timeout -s KILL 300 python tools/profile_solve.py "$@" 2>&1 | tail -1 | cut -c1-70)"
done
done
