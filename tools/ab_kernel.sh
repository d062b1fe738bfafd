#!/bin/bash
# Same-box A/B of one kernel's duration under ncu (dev tool): ab_kernel.sh REGEX [profile_solve args]
cd "$(dirname "$0")/.."
re=$1; shift
for lib in base new; do
  if [ $lib = base ]; then export KNN_B200_LIB=$PWD/paper_0906_0231_b200/lib/libknn_b200_base.so; else unset KNN_B200_LIB; fi
  timeout -s KILL 600 ncu -k "regex:$re" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file /tmp/abk_$lib.csv python tools/profile_solve.py "$@" > /dev/null 2>&1
  echo "$lib $(python tools/launch_summary.py /tmp/abk_$lib.csv | head -3)"
done
