"""Probe: GPU apply vs the unmodified reference (oracle/_ref RefRaw) on the
same SBDOPv1 file at a BASELINE config size; prints timings and rel l2.

  python tools/ref_scale.py --config 4 [--scale 1.0]
"""
import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1711_07877_b200 as sbd  # noqa: E402
from oracle.oracle import RefLib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--scale", type=float, default=1.0)
args = ap.parse_args()
w = bench.workload(args.config, args.scale)
z = w["z"]
n = len(z)
t0 = time.perf_counter()
dmax = sbd.cloud_diameter(z)
kern = sbd.kernel_helmholtz(w["kappa"] / dmax) if w["kind"] else sbd.kernel_laplace()
a = w["dmin"] / dmax if w["dmin"] else 0.0
op = sbd.CompressedOperator.assemble(kern, z, opts=sbd.AssembleOptions(eps=w["eps"], a_override=a,
                                                                        max_grid_bytes=96 << 30))
print(f"assemble {time.perf_counter() - t0:.1f}s info {op.info()}", flush=True)
path = f"/tmp/ref_scale_{os.getpid()}.sbdop"
op.save(path)
f = bench.rhs(w, n, np.random.default_rng(5))
q = op.apply(f)
t0 = time.perf_counter()
raw = RefLib().raw(path, max_grid_bytes=96 << 30)
t_open = time.perf_counter() - t0
t0 = time.perf_counter()
q_ref = raw.apply(f, n)
t_apply = time.perf_counter() - t0
rel = float(np.linalg.norm(q - q_ref) / np.linalg.norm(q_ref))
relre = float(np.linalg.norm(q.real - q_ref.real) / np.linalg.norm(q_ref))
print(f"config {args.config} N={n}: ref open {t_open:.1f}s apply {t_apply:.1f}s; rel_l2 {rel:.3e} (real part {relre:.3e})",
      flush=True)
os.unlink(path)
