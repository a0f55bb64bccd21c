#!/bin/bash
# One ncu --set full capture of a kernel of tests/sweep_variants.py (run on a
# B200 via gpurun):  bash profiles/ncu_one.sh <tag> <config> <variant> <kernel-regex>
set -u
TAG=$1; CFG=$2; VAR=$3; K=$4
mkdir -p gpurun_out
python tests/sweep_variants.py --config $CFG --variants=$VAR --iters 3 > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/$TAG \
    python tests/sweep_variants.py --config $CFG --variants=$VAR --iters 3 > gpurun_out/${TAG}_ncu.log 2>&1
tail -1 gpurun_out/${TAG}_ncu.log
