"""Time the complex pipeline on a real-f workload's operator (a complex f; dev tool)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1711_07877_b200 as sbd  # noqa: E402

w = bench.workload("4", 1.0)
z = w["z"]
d = sbd.cloud_diameter(z)
ik = sys.argv[1] if len(sys.argv) > 1 else "auto"
op = sbd.CompressedOperator.assemble(
    sbd.kernel_laplace(), z, opts=sbd.AssembleOptions(eps=w["eps"], a_override=w["dmin"] / d, max_grid_bytes=96 << 30,
                                                      pipeline=sbd.OpOptions(interp_kernel=ik)))
rng = np.random.default_rng(1)
n = len(z)
fc = (rng.standard_normal(n) + 1j * rng.standard_normal(n))
fd = torch.from_numpy(fc.view(np.float64).copy()).cuda()
qd = torch.empty_like(fd)
op.set_profiling(True)
for _ in range(3):
    op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, 0, f_is_real=False)
torch.cuda.synchronize()
op.stage_times()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, 0, f_is_real=False)
e1.record()
torch.cuda.synchronize()
agg = {}
for nm, ms in op.stage_times():
    agg[nm] = agg.get(nm, 0.0) + ms / 5
print({"interp_kernel": ik, "complex_ms_per_apply": e0.elapsed_time(e1) / 5, "stages": {k: round(v, 3) for k, v in agg.items()}})
