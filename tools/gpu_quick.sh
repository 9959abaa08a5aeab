python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/t1.log 2>&1; echo tests=$?; tail -3 gpurun_out/t1.log; python bench.py --ref-full 0 --steps 10 --warmup 3 > gpurun_out/bench1.log 2>gpurun_out/bench1.err; echo bench=$?; python - <<EOP
import json
l=[x for x in open("gpurun_out/bench1.log") if x.startswith("{")][-1]
d=json.loads(l)
print(d["ms_per_step"], d["roofline"]["stages_ms"], d["adjoint"], d["config"]["offline_s"])
EOP
tail -3 gpurun_out/bench1.err
