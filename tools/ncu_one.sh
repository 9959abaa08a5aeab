#!/bin/bash
# ncu --set full of one launch of a kernel in tools/prof_apply.py (dev tool)
#   tools/ncu_one.sh <kernel regex> <launch-skip> <out name>
cd "$(dirname "$0")/.."
ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 --launch-count 1 \
    -o gpurun_out/$3 python tools/prof_apply.py --applies 2 > gpurun_out/ncu_$3.log 2>&1
echo ncu=$?
