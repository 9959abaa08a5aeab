#!/bin/bash
# launch list + --set full of the hot kernels of one config-4 apply (dev tool;
# summarised into profiles/ by tools/ncu_summary.py)
cd "$(dirname "$0")/.."
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches.csv python tools/prof_apply.py --applies 3 > gpurun_out/ncu_launch.log 2>&1
echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"k_interp_tile|k_interp_real|k_spread_cta|k_spmv_vec" \
    --launch-skip 5 --launch-count 5 -o gpurun_out/hot python tools/prof_apply.py --applies 2 > gpurun_out/ncu_hot.log 2>&1
echo hot=$?
