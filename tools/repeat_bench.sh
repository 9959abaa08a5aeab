#!/bin/bash
# run the short config-4 bench N times in fresh processes and print the stage times (dev tool)
cd "$(dirname "$0")/.."
for i in $(seq 1 ${1:-6}); do
  python bench.py --ref-full 0 --no-cpu-baseline --adjoint 0 --procedural 0 --nrhs 1 --steps 10 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['roofline']['stages_ms']; print(round(d['ms_per_step'],3), s['spread_src'], s['spmv'], s['spread_xi'], s['interp_tgt'])"
done
