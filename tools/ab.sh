#!/bin/bash
# A/B kernel variants on one GPU box: rebuild the library with each set of
# extra nvcc flags (in this scratch copy of the tree) and time the kernels.
#   bash tools/ab.sh "cfgs" "FLAGS_A" "FLAGS_B" ...
cd "$(dirname "$0")/.."
CFGS=$1; shift
for V in "$@"; do
    make -s -C paper_2108_07031_b200/csrc clean >/dev/null
    make -s -C paper_2108_07031_b200/csrc NVEXTRA="$V" > /dev/null 2>&1 || { echo "build failed: $V"; continue; }
    for C in $CFGS; do
        echo -n "[$V] "
        python tools/kperf.py $C 10 2>/dev/null | tail -1
    done
done
