#!/bin/bash
# Same-box A/B of an environment knob (dev tool): ab_knob.sh VAR VAL_A VAL_B [profile_solve args]
cd "$(dirname "$0")/.."
var=$1 a=$2 b=$3; shift 3
for v in $a $b $a $b; do
  echo "$var=$v $(env $var=$v timeout -s KILL 300 python tools/profile_solve.py "$@" 2>&1 | tail -1 | cut -c1-140)"
done
