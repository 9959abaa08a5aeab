"""Time one config's apply with stored arrays vs procedural ring nodes (dev tool)."""
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
fd = torch.from_numpy(f.view(np.float64).copy()).cuda()
out = {}
for proc in (False, True):
    op = sbd.CompressedOperator.assemble(
        kern, z, opts=sbd.AssembleOptions(eps=w["eps"], a_override=(w["dmin"] / d if w["dmin"] else 0.0),
                                          max_grid_bytes=96 << 30,
                                          pipeline=sbd.OpOptions(procedural_rings=proc, verbose=proc)))
    qd = torch.empty_like(fd)
    for _ in range(3):
        op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, 0, f_is_real=not w["f_complex"])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, 0, f_is_real=not w["f_complex"])
    e1.record()
    torch.cuda.synchronize()
    info = op.info()
    out[proc] = (e0.elapsed_time(e1) / 10, info["device_bytes"], info["procedural_rings"], qd.cpu().numpy().copy())
    del op
    torch.cuda.empty_cache()
rel = np.linalg.norm(out[True][3] - out[False][3]) / np.linalg.norm(out[False][3])
print({"stored_ms": out[False][0], "procedural_ms": out[True][0], "stored_bytes": out[False][1],
       "procedural_bytes": out[True][1], "procedural_on": out[True][2], "rel_l2": rel})
