"""Do two applies on two streams overlap (HBM-bound FFT passes beside the
issue-bound spread / interpolation kernels)? Two operators of the same
workload, applied back to back on one stream vs concurrently on two (dev tool)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1711_07877_b200 as sbd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
w = bench.workload(a.config, a.scale)
z = w["z"]
d = sbd.cloud_diameter(z)
kern = sbd.kernel_helmholtz(w["kappa"] / d) if w["kind"] else sbd.kernel_laplace()
f = bench.rhs(w, len(z), np.random.default_rng(1))
ops = [sbd.CompressedOperator.assemble(
    kern, z, opts=sbd.AssembleOptions(eps=w["eps"], a_override=(w["dmin"] / d if w["dmin"] else 0.0),
                                      max_grid_bytes=96 << 30)) for _ in range(2)]
fd = torch.from_numpy(f.view(np.float64).copy()).cuda()
qd = [torch.empty_like(fd) for _ in range(2)]
st = [torch.cuda.Stream(), torch.cuda.Stream()]
real = not w["f_complex"]


def run(two_streams, reps=10):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in st:
        s.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        for i in range(2):
            s = st[i if two_streams else 0]
            ops[i].apply_device(fd.data_ptr(), qd[i].data_ptr(), 1, s.cuda_stream, f_is_real=real)
    for s in st:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (2 * reps)


run(False, 2)
run(True, 2)
print({"one_stream_ms_per_apply": run(False), "two_streams_ms_per_apply": run(True)})
