#!/bin/bash
# Same-box A/B of tools/ab_build.sh's two libraries (dev tool): ab_time.sh [profile_solve args]
cd "$(dirname "$0")/.."
for lib in base new base new; do
  if [ $lib = base ]; then export KNN_B200_LIB=$PWD/paper_0906_0231_b200/lib/libknn_b200_base.so; else unset KNN_B200_LIB; fi
  echo "$lib $(timeout -s KILL 300 python tools/profile_solve.py "$@" 2>&1 | tail -1 | cut -c1-60)"
done
