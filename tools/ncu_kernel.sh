#!/bin/bash
# One ncu --set full capture (source-level stalls) of one kernel launch of a
# bench step: bash tools/ncu_kernel.sh <config> <kernel regex> <skip> <tag>
cd "$(dirname "$0")/.."
CFG=$1; K=$2; SKIP=${3:-2}; TAG=${4:-cap}
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$K" --launch-skip $SKIP -c 1 -f \
    -o /tmp/$TAG python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/$TAG.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_sass.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_sass.csv
ls -la gpurun_out/${TAG}*
