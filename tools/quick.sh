#!/bin/bash
# dev loop on the GPU box: gpu tests + one bench line (stage times)
cd "$(dirname "$0")/.."
if [ "$1" != "notest" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
fi
for v in ${SPREADS:-l}; do
  SBD_SPREAD=$v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$v.log 2>&1; echo bench=$?
  tail -1 gpurun_out/bench_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['stages_ms'])"
done
