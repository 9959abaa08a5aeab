"""Time the product's offline assembly for a bench config (dev tool)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_1711_07877_b200 as sbd
w = bench.workload(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0)
z = w["z"]; d = sbd.cloud_diameter(z)
kern = sbd.kernel_helmholtz(w["kappa"] / d) if w["kind"] else sbd.kernel_laplace()
t = time.time()
op = sbd.CompressedOperator.assemble(kern, z, opts=sbd.AssembleOptions(eps=w["eps"], a_override=(w["dmin"] / d if w["dmin"] else 0.0), max_grid_bytes=96 << 30))
print("assemble", time.time() - t, op.info()["P"], op.info()["n_xi"], op.info()["nnz"])
