#!/bin/bash
# Build the committed HEAD library as paper_0906_0231_b200/lib/libknn_b200_base.so
# next to the working-tree build, for same-box A/B timing (dev tool).
set -e
cd "$(dirname "$0")/.."
git stash -q
make -j8 lib >/dev/null 2>&1 || { git stash pop -q; exit 1; }
cp paper_0906_0231_b200/lib/libknn_b200.so /tmp/libknn_b200_base.so
git stash pop -q
make -j8 lib >/dev/null 2>&1
cp /tmp/libknn_b200_base.so paper_0906_0231_b200/lib/libknn_b200_base.so
echo "built base (HEAD) and working tree"
