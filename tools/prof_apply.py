"""Profiling driver (not part of the product): assemble a bench workload and
run a few applies, for ncu launch lists / kernel captures."""
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
ap.add_argument("--applies", type=int, default=3)
ap.add_argument("--verbose", type=int, default=0)
a = ap.parse_args()
w = bench.workload(a.config, a.scale)
z = w["z"]
d = sbd.cloud_diameter(z)
kern = sbd.kernel_helmholtz(w["kappa"] / d) if w["kind"] else sbd.kernel_laplace()
op = sbd.CompressedOperator.assemble(
    kern, z, opts=sbd.AssembleOptions(eps=w["eps"], a_override=(w["dmin"] / d if w["dmin"] else 0.0),
                                      max_grid_bytes=96 << 30,
                                      pipeline=sbd.OpOptions(verbose=bool(a.verbose))))
f = bench.rhs(w, len(z), np.random.default_rng(1))
fd = torch.from_numpy(f.view(np.float64).copy()).cuda()
qd = torch.empty_like(fd)
for _ in range(a.applies):
    op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, 0, f_is_real=not w["f_complex"])
torch.cuda.synchronize()
print("ok", op.info()["n_xi"])
