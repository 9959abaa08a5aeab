"""Slab decomposition at a BASELINE size with G ranks emulated on one B200
(dev tool): every rank's three stages are timed separately with CUDA events,
the all-to-alls are device copies (their byte counts are reported), and the
assembled q is checked against the single-device complex apply.

  python tools/slab_model.py [--config 4] [--world 8] [--reps 3]

Prints one JSON line: per-stage max-over-ranks times, exchange bytes per rank,
and the predicted G-GPU apply time (stage maxima + exchanges at an assumed
all-to-all bandwidth per GPU)."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_1711_07877_b200 as sbd  # noqa: E402
from paper_1711_07877_b200.parallel import SlabApply  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--a2a-gbs", type=float, default=700.0, help="assumed all-to-all GB/s per GPU (NVLink 5)")
args = ap.parse_args()
w = bench.workload(args.config)
z = w["z"]
n = len(z)
dmax = sbd.cloud_diameter(z)
kern = sbd.kernel_helmholtz(w["kappa"] / dmax) if w["kind"] else sbd.kernel_laplace()
a = w["dmin"] / dmax if w["dmin"] else w.get("a", 0.0)
op = sbd.CompressedOperator.assemble(kern, z, opts=sbd.AssembleOptions(
    eps=w["eps"], a_override=a, max_grid_bytes=96 << 30))
f_np = bench.rhs(w, n, np.random.default_rng(1))
f = torch.from_numpy(f_np.view(np.float64).copy()).cuda()
q = torch.zeros(2 * n, dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
G = args.world
ranks = [SlabApply(op, r, G, alltoall=lambda *x: None) for r in range(G)]
t_build = time.perf_counter() - t0


def exchange(e):
    for r, dst in enumerate(ranks):
        recv = dst.bufs[e][1]
        ro = 0
        for k, src in enumerate(ranks):
            ssp = src.splits[e][0]
            so = sum(ssp[:r])
            m = ssp[r]
            recv[ro:ro + m].copy_(src.bufs[e][0][so:so + m])
            ro += m


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


stage_ms = np.zeros((args.reps, 3, G))
for rep in range(args.reps + 1):
    q.zero_()
    for r, s in enumerate(ranks):
        ms = timed(lambda: s.stage(0, None, f, s.bufs[0][0]))
        if rep:
            stage_ms[rep - 1, 0, r] = ms
    exchange(0)
    for r, s in enumerate(ranks):
        ms = timed(lambda: s.stage(1, s.bufs[0][1], None, s.bufs[1][0]))
        if rep:
            stage_ms[rep - 1, 1, r] = ms
    exchange(1)
    for r, s in enumerate(ranks):
        ms = timed(lambda: s.stage(2, s.bufs[1][1], f, q))
        if rep:
            stage_ms[rep - 1, 2, r] = ms
torch.cuda.synchronize()
qs = q.cpu().numpy().view(np.complex128)
# the single-device apply of the same f (for a real f the default operator's
# half split drops the ~1e-10 imaginary parts the complex slab path keeps)
fd = torch.from_numpy(f_np.view(np.float64).copy()).cuda()
qd = torch.empty(2 * n, dtype=torch.float64, device="cuda")
op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, 0)
torch.cuda.synchronize()
qref = qd.cpu().numpy().view(np.complex128)
rel = float(np.linalg.norm(qs - qref) / np.linalg.norm(qref))
med = np.median(stage_ms, axis=0)  # (stage, rank)
per_stage_max = med.max(axis=1)
x_bytes = [max(16 * sum(s.splits[e][0]) // 2 for s in ranks) for e in (0, 1)]
x_ms = [b / (args.a2a_gbs * 1e9) * 1e3 for b in x_bytes]
pred = float(per_stage_max.sum() + sum(x_ms))
print(json.dumps({
    "config": args.config, "N": n, "world": G, "build_s": round(t_build, 1),
    "stage_ms_max_over_ranks": [round(float(x), 3) for x in per_stage_max],
    "stage_ms_by_rank": [[round(float(x), 3) for x in row] for row in med],
    "exchange_bytes_per_rank_max": x_bytes, "exchange_ms_at_%dGBs" % int(args.a2a_gbs): [round(x, 3) for x in x_ms],
    "predicted_ms_per_apply": round(pred, 3), "predicted_points_per_s": n / (pred / 1e3),
    "rel_l2_vs_single_device": rel,
}), flush=True)
