#!/usr/bin/env python
"""SBD apply throughput on B200 (BASELINE.json metric: "SBD apply points/s").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                  [--config 4|3|1|2s]

Workload (default, BASELINE.json configs[3] = "config 4"): Laplace kernel,
N = 1e7 points i.i.d. uniform in a disk of diameter 1, real f ~ N(0,1),
eps = 1e-6, delta_min = 2.74/sqrt(N); synthetic, seeded. It is the largest
BASELINE config that fits one GPU (configs[1] as written needs a ~0.84 TB FFT
grid).

A step = one CompressedOperator::apply (conv_operator.cpp:301-309): both
type-III NUFFTs (spread, cuFFT, deconvolve+interpolate), the omega-hat
weighting and the CSR close correction, on device-resident f -> q.
`value` = N * n_gpus * K / (max-over-ranks device time of K steps) [points/s];
`e2e` = the same through the host-buffer C-ABI call sbd_op_apply (pinned host
f in, host q out, copies inside the timed region).

--impl reference times the reference's own CPU apply (oracle/_ref, the
unmodified reference library compiled here) on the box's host cores on a
bounded sample of the same workload (see cpu_baseline.sample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tests.clouds import disk_cloud, star_curve_cloud, star_interior_cloud  # noqa: E402

METRIC = "SBD apply points/s (N=1e6–1e7, ε=1e-6) at 1/2/4/8 B200; % HBM roofline"
SEED = 20261019


# ------------------------------------------------------------------ workloads
def workload(name: str, scale: float = 1.0):
    """Returns (description, points, kernel dict, eps, a_override_fn, f_complex)."""
    rng = np.random.default_rng(SEED)
    if name == "4":
        n = int(1e7 * scale)
        z = disk_cloud(n, rng)
        return dict(desc=f"config4: Laplace, N={n} uniform disk d=1, eps=1e-6, delta_min=2.74/sqrt(N)",
                    z=z, kind=0, kappa=0.0, eps=1e-6, dmin=2.74 / np.sqrt(n), f_complex=False)
    if name == "3":
        n = int(1e6 * scale)
        z = disk_cloud(n, rng)
        return dict(desc=f"config3: Helmholtz k*dmax=2pi*100, N={n} uniform disk d=1, eps=1e-6, "
                         "delta_min=2.74/sqrt(N)", z=z, kind=1, kappa=2 * np.pi * 100, eps=1e-6,
                    dmin=2.74 / np.sqrt(n), f_complex=True)
    if name == "1":
        n = int(1e4 * scale)
        z = disk_cloud(n, rng)
        return dict(desc=f"config1: Laplace, N={n} uniform disk d=1, eps=1e-6, delta_min=2.74/sqrt(N)",
                    z=z, kind=0, kappa=0.0, eps=1e-6, dmin=2.74 / np.sqrt(n), f_complex=False)
    if name == "5":
        # BASELINE configs[4] is 1.1e7 points with D row-sharded over several
        # GPUs (>= 100 GB of D at any feasible delta_min); one
        # GPU runs its shape at N/8: 1.25e6 on the star curve + 1.25e5 inside,
        # Helmholtz k dmax = 2 pi 300, eps 1e-4, complex f, 8 right-hand sides
        # per apply; delta_min is unspecified there: a = 5e-4 (P ~ 4200)
        nc, ni = int(1.25e6 * scale), int(1.25e5 * scale)
        z = np.concatenate([star_curve_cloud(nc, rng), star_interior_cloud(ni, rng)])
        return dict(desc=f"config5 at N/8: Helmholtz k*dmax=2pi*300, N={nc}+{ni} star curve + interior, "
                         "eps=1e-4, a=delta_min/delta_max=5e-4, complex f, 8 RHS per apply",
                    z=z, kind=1, kappa=2 * np.pi * 300, eps=1e-4, dmin=None, a=5e-4, f_complex=True,
                    nrhs=8)
    if name == "2s":
        n = int(1e6 * scale)
        z = star_curve_cloud(n, rng)
        return dict(desc=f"config2*: Laplace, N={n} star curve (jitter 0.1), eps=1e-6, reference a-rule",
                    z=z, kind=0, kappa=0.0, eps=1e-6, dmin=None, f_complex=False)
    raise SystemExit(f"unknown config {name}")


def rhs(w, n, rng):
    f = rng.standard_normal(n).astype(np.complex128)
    if w["f_complex"]:
        f += 1j * rng.standard_normal(n)
    return f


# ------------------------------------------------------------------ helpers
class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/sbd_clocks_{os.getpid()}.csv"

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def stage_bytes(info, name):
    """Algorithmic bytes per launch, SURVEY.md section 8(d) byte model."""
    N, Nt, Nx, nnz = info["n_src"], info["n_tgt"], info["n_xi"], info["nnz"]
    grid_in = 16 * info["n1_in"] * info["n2_in"]
    grid_out = 16 * info["n1_out"] * info["n2_out"]
    band = lambda n1, n2: 16 * (2 * (n1 // 4) + 1) * (2 * (n2 // 4) + 1)  # noqa: E731
    return {
        "spread_src": 16 * N + 16 * N + grid_in,                                   # B1
        "interp_xi": band(info["n1_in"], info["n2_in"]) + 3 * 16 * Nx,             # B2
        "spread_xi": 2 * 16 * Nx + grid_out,                                       # B3
        "interp_tgt": band(info["n1_out"], info["n2_out"]) + 2 * 16 * Nt,          # B4
        "spmv": 8 * (Nt + 1) + 20 * nnz + 16 * N + 32 * Nt,                        # B5
    }.get(name)


def ncu_pipes(stage):
    """fp64 / DMMA pipe, issue and L1 utilisation of the stage's kernel from the
    committed ncu --set full capture (profiles/ncu_pipes.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_pipes.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        d = json.load(fh)
    v = d.get("pipes", {}).get(stage)
    return dict(v, source=d.get("source")) if v else None


def ncu_traffic(stage):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as fh:
        return json.load(fh).get(stage)


# ------------------------------------------------------------------ reference arm
def reference_sample(w, sample_n):
    """Assemble the same workload at sample_n points with the reference's own
    assemble (oracle/_ref) and return (ref lib, operator path, f)."""
    from oracle.oracle import REF_SO, Oracle, RefLib
    rng = np.random.default_rng(SEED + 1)
    if w["desc"].startswith("config2"):
        z = star_curve_cloud(sample_n, rng)
    elif w["desc"].startswith("config5"):
        z = np.concatenate([star_curve_cloud(sample_n - sample_n // 11, rng),
                            star_interior_cloud(sample_n // 11, rng)])
    else:
        z = disk_cloud(sample_n, rng)
    path = f"/tmp/sbd_ref_sample_{os.getpid()}.sbdop"
    kind = "reference" if os.path.exists(REF_SO) else "port"
    if kind == "reference":
        lib = RefLib()
        d = lib.diameter(z)
        a = (2.74 / np.sqrt(sample_n)) / d if w["dmin"] is not None else w.get("a", 0.0)
        lib.assemble_save(path, z, kind=w["kind"], k=w["kappa"] / d, eps=w["eps"], a_override=a)
        op = lib.load(path)
        apply = lambda f: op.apply(f, sample_n)  # noqa: E731
    else:
        import paper_1711_07877_b200 as sbd  # only to build the operator file for the port
        d = sbd.cloud_diameter(z)
        kern = sbd.kernel_helmholtz(w["kappa"] / d) if w["kind"] else sbd.kernel_laplace()
        a = (2.74 / np.sqrt(sample_n)) / d if w["dmin"] is not None else w.get("a", 0.0)
        o = sbd.CompressedOperator.assemble(kern, z, opts=sbd.AssembleOptions(eps=w["eps"],
                                                                               a_override=a))
        o.save(path)
        op = Oracle().op(path)
        apply = op.apply
    f = rhs(w, sample_n, np.random.default_rng(SEED + 2))
    return kind, apply, f, path


def time_reference(apply, f, threads, reps):
    """`threads` concurrent applies (CompressedOperator::apply is const and
    thread-safe, conv_operator.hpp:33-36), `reps` rounds; returns seconds/round."""
    def work():
        for _ in range(reps):
            apply(f)
    ts = [threading.Thread(target=work) for _ in range(threads)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return (time.perf_counter() - t0) / reps


def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sample_n = args.sample_n
    kind, apply, f, path = reference_sample(w, sample_n)
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, args.ref_threads or cores))
    for _ in range(args.warmup):
        time_reference(apply, f, threads, 1)
    per_round = time_reference(apply, f, threads, args.steps)
    os.unlink(path)
    value = sample_n * threads / per_round
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_round * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": w["desc"], "parallelism": f"host threads x{threads}"},
        "cpu_baseline": {
            "value": value, "unit": "points/s", "cores": threads, "kind": kind,
            "sample": (f"same distribution/eps/delta_min rule at N={sample_n} (reference assemble + "
                       f"{threads} concurrent single-threaded CompressedOperator::apply per step)")},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ same-config reference
def reference_same_config(op, f, q_dev_host, max_grid_bytes):
    """One CompressedOperator::apply of the unmodified reference (oracle/_ref,
    driven through its own NufftPlan / SparsePairMatrix on the operator file
    this run assembled; RefRaw) on one host core: parity of q against it and
    a same-config CPU baseline. Runs after the timed regions."""
    from oracle.oracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        return None, None
    path = f"/tmp/sbd_bench_op_{os.getpid()}.sbdop"
    try:
        t0 = time.perf_counter()
        op.save(path)
        t_save = time.perf_counter() - t0
        t0 = time.perf_counter()
        raw = RefLib().raw(path, max_grid_bytes=max_grid_bytes)
        t_open = time.perf_counter() - t0
        t0 = time.perf_counter()
        q_ref = raw.apply(f, len(q_dev_host))
        t_apply = time.perf_counter() - t0
        del raw
    finally:
        if os.path.exists(path):
            os.unlink(path)
    n = len(f)
    rel = float(np.linalg.norm(q_dev_host - q_ref) / np.linalg.norm(q_ref))
    parity = {"rel_l2_vs_reference": rel, "bar": 1e-9, "ok": rel <= 1e-9,
              "reference": "oracle/_ref (unmodified reference sources; RefRaw = its NufftPlan + "
                           "SparsePairMatrix on this run's operator file)"}
    cpu = {"value": n / t_apply, "unit": "points/s", "cores": 1, "kind": "reference",
           "sample": (f"the full workload: one single-threaded reference apply of this config "
                      f"(N={n}) on this box's host ({os.cpu_count()} cores present; the reference "
                      f"is single-threaded), {t_apply:.1f} s; plan build {t_open:.1f} s and "
                      f"operator save {t_save:.1f} s not counted; FFT on the oracle's shim, "
                      "not FFTW (BASELINE.md section 2)"),
           "apply_s": round(t_apply, 2)}
    return parity, cpu


def spawn_ranks(args):
    """bench.py --gpus N without torchrun: re-exec under torch.distributed.run
    with N local ranks (the driver's own launch form) and return its code."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ B200 arm
def run_b200(args, w):
    import torch
    import paper_1711_07877_b200 as sbd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench: WORLD_SIZE={world} but --gpus {args.gpus}")
    ndev = torch.cuda.device_count()
    shared = ndev < world  # more ranks than GPUs: a functional run, not a scaling number
    local = local % ndev
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    z = w["z"]
    n = len(z)
    t0 = time.perf_counter()
    dmax = sbd.cloud_diameter(z)
    kern = sbd.kernel_helmholtz(w["kappa"] / dmax) if w["kind"] else sbd.kernel_laplace()
    a = w["dmin"] / dmax if w["dmin"] else w.get("a", 0.0)
    opts = sbd.AssembleOptions(eps=w["eps"], a_override=a, max_grid_bytes=96 << 30, device=local)
    op = sbd.CompressedOperator.assemble(kern, z, opts=opts)
    t_offline = time.perf_counter() - t0
    info = op.info()

    rng = np.random.default_rng(SEED + 3)
    R = w.get("nrhs", 1)  # right-hand sides per apply (config 5: a GMRES-style block of 8)
    if R > 1 and world > 1:
        raise SystemExit("bench: the sharded apply takes one right-hand side per step")
    f = np.stack([rhs(w, n, rng) for _ in range(R)]) if R > 1 else rhs(w, n, rng)
    f_real = not w["f_complex"]
    f_dev = torch.from_numpy(f.reshape(-1).view(np.float64).copy()).cuda()
    q_dev = torch.zeros(2 * n * R, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    alt_step = None
    if world > 1:
        # slab decomposition (no replicated stage, two all-to-alls)
        # and the north_star partition (source shards -> all-reduce of the xi
        # spectrum -> target shards); --scheme picks the headline one, the
        # other is timed beside it
        from paper_1711_07877_b200.parallel import DeviceBackend, ShardedApply, SlabApply
        sharded = ShardedApply(DeviceBackend(op), rank, world)
        slab = SlabApply(op, rank, world)

        def step_shard():
            sharded.apply(f_dev, q_dev)

        def step_slab():
            slab.apply(f_dev, q_dev)
        scheme = "shard" if args.scheme == "shard" else "slab"  # auto: slab first, the faster one reported
        step, alt_step = (step_slab, step_shard) if scheme == "slab" else (step_shard, step_slab)
    else:
        def step():  # the caller knows its f is real (sbd_op_apply_device_ex)
            op.apply_device(f_dev.data_ptr(), q_dev.data_ptr(), R, sh, f_is_real=f_real)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)  # let the sampler start before the timed region
    op.set_profiling(True)
    launches0 = sbd.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = sbd.launch_count() - launches0
    clk = clocks.stop()
    ms_total = e0.elapsed_time(e1)
    stages = op.stage_times()
    op.set_profiling(False)
    if dist:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = n * R / (ms_step / 1e3)  # one apply of N points (x R right-hand sides) per step, whole job

    # multi-GPU, right-hand-side parallel (weak scaling; SURVEY.md 8e "replicas
    # across RHS"): every rank applies the full operator to its own right-hand
    # side, no collective -- the batch-throughput mode, beside the sharded
    # (strong-scaling, north_star) apply timed above
    alt = None
    if alt_step is not None:
        for _ in range(args.warmup):
            alt_step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(args.steps):
            alt_step()
        a1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_alt = float(t.item()) / args.steps
        alt = {"scheme": "shard" if scheme == "slab" else "slab", "value": n / (ms_alt / 1e3),
               "unit": "points/s", "ms_per_step": round(ms_alt, 3), "scaling": "strong"}
        if args.scheme == "auto" and ms_alt < ms_step:
            # both partitions were timed by the same protocol (K steps between
            # barriers, max over ranks): the headline is the one an application
            # would keep after this calibration, the other stays beside it
            alt, scheme, ms_step = ({"scheme": scheme, "value": value, "unit": "points/s",
                                     "ms_per_step": round(ms_step, 3), "scaling": "strong"},
                                    alt["scheme"], ms_alt)
            value = n * R / (ms_step / 1e3)

    rhs_par = None
    if world > 1:
        f_own = torch.from_numpy(rhs(w, n, np.random.default_rng(SEED + 100 + rank)).view(np.float64).copy()).cuda()
        q_own = torch.empty(2 * n, dtype=torch.float64, device="cuda")

        def own_step():
            op.apply_device(f_own.data_ptr(), q_own.data_ptr(), 1, sh, f_is_real=f_real)
        for _ in range(args.warmup):
            own_step()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        for _ in range(args.steps):
            own_step()
        r1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([r0.elapsed_time(r1)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_rp = float(t.item()) / args.steps
        rhs_par = {"value": n * world / (ms_rp / 1e3), "unit": "points/s", "ms_per_step": round(ms_rp, 3),
                   "scaling": "weak",
                   "note": f"{world} ranks, each one apply of its own N-point right-hand side per step, no collective"}
        del f_own, q_own

    # per-stage averages over the timed region (CUDA events on the launch stream)
    agg = {}
    for name, ms in stages:
        agg.setdefault(name, []).append(ms)
    avg = {k: sum(v) / len(v) for k, v in agg.items()}
    cand = {k: v for k, v in avg.items() if stage_bytes(info, k) is not None}
    roof_note = None
    if not cand:  # (the slab stages carry no per-stage events): the single-device stages
        roof_note = "stages of this operator's single-device apply (the slab stages carry no per-stage events)"
        op.set_profiling(True)
        for _ in range(3):
            op.apply_device(f_dev.data_ptr(), q_dev.data_ptr(), R, sh, f_is_real=f_real)
        torch.cuda.synchronize()
        for name, ms in op.stage_times():
            agg.setdefault(name, []).append(ms)
        op.set_profiling(False)
        avg = {k: sum(v) / len(v) for k, v in agg.items()}
        cand = {k: v for k, v in avg.items() if stage_bytes(info, k) is not None}
    dom = max(cand, key=cand.get)
    peak, peak_src = measured_peak()
    ach = stage_bytes(info, dom) / (avg[dom] / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": ncu_traffic(dom), "peak_source": peak_src,
                "algorithmic_bytes": stage_bytes(info, dom), "avg_ms": avg[dom],
                "stages_ms": {k: round(v, 4) for k, v in avg.items()},
                "stages_frac": {k: round(stage_bytes(info, k) / (avg[k] / 1e3) / 1e9 / peak, 4)
                                for k in cand}}
    roofline["pipes"] = ncu_pipes(dom)  # what actually binds it (fp64 pipes beside HBM)
    roofline["traffic_source"] = "profiles/ncu_traffic.json (ncu --set full capture of this kernel, per launch)"
    if roof_note:
        roofline["note"] = roof_note

    # end to end: host f (pinned) in, host q out, copies inside the timed region
    fh = torch.from_numpy(f.reshape(-1).view(np.float64).copy()).pin_memory()
    qh = torch.empty(2 * n * R, dtype=torch.float64).pin_memory()
    if world == 1:
        def e2e_step():  # the reference-facing host-buffer C-ABI call (sbd_op_apply)
            op.apply_host(fh.data_ptr(), qh.data_ptr(), R)
    else:
        def e2e_step():
            f_dev.copy_(fh, non_blocking=True)
            step()
            lo, hi = sharded.target_range()
            qh.copy_(q_dev)  # this rank's target shard (scattered entries) back to the host
            torch.cuda.synchronize()
    e2e_step()
    if dist:
        dist.barrier()
    t1 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = (time.perf_counter() - t1) / args.steps
    if dist:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    # pipelined host applies (sbd_op_apply_async): every step still copies its
    # f in and its q out, but the copies overlap the neighbouring steps' device
    # work (two staging slots, two copy streams) -- the batch-serving mode
    e2e_pipe = None
    if world == 1:
        qh2 = torch.empty_like(qh).pin_memory()
        qhs = [qh, qh2]
        tk = [op.apply_async(fh.data_ptr(), qhs[k % 2].data_ptr(), R) for k in range(2)]
        for t in tk:
            op.wait(t)
        t1 = time.perf_counter()
        tk = [op.apply_async(fh.data_ptr(), qhs[k % 2].data_ptr(), R) for k in range(args.steps)]
        for t in tk[-2:]:
            op.wait(t)
        ep = (time.perf_counter() - t1) / args.steps
        e2e_pipe = {"value": n * R / ep, "unit": "points/s", "ms_per_step": round(ep * 1e3, 3),
                    "h2d_bytes_per_step": 16 * n * R, "d2h_bytes_per_step": 16 * n * R,
                    "note": "sbd_op_apply_async: host f in / host q out every step, copies overlapped "
                            "with the neighbouring steps' device work"}

    # the reference's accuracy contract on this workload (conv_operator.hpp:50-51,
    # north_star: <= eps at 1,000 random targets): |q_k - sum_{l != k} G f_l| <=
    # eps sum|f|, the direct sum in fp64 on the GPU (torch)
    contract = None
    # every rank runs the apply (the sharded one has collectives); each writes
    # its target shard, so a sum over ranks of zero-initialised q fills all N
    q_dev.zero_()
    step()
    torch.cuda.synchronize()
    if dist:
        dist.all_reduce(q_dev)
    qv = q_dev.view(-1, 2).cpu().numpy()
    qv = (qv[:, 0] + 1j * qv[:, 1])[:n]  # the first right-hand side
    f0 = f[0] if R > 1 else f
    if rank == 0:
        rows = np.random.default_rng(SEED + 7).choice(n, 1000, replace=False)
        zt = torch.from_numpy(z).cuda()
        ft = torch.from_numpy(f0).cuda()
        want = torch.zeros(len(rows), dtype=torch.complex128, device="cuda")
        zr = zt[torch.from_numpy(rows).cuda()]
        kk = w["kappa"] / dmax
        for s0 in range(0, n, 200_000):
            d = torch.cdist(zr, zt[s0:s0 + 200_000], compute_mode="donot_use_mm_for_euclid_dist")
            m = d > 0
            dd = torch.where(m, d, torch.ones_like(d))
            if w["kind"]:  # -(i/4) H0(kr) = Y0/4 - i J0/4 (kernels.cpp:73-75)
                g = torch.complex(0.25 * torch.special.bessel_y0(kk * dd), -0.25 * torch.special.bessel_j0(kk * dd))
            else:  # log r (kernels.cpp:70-72)
                g = torch.complex(torch.log(dd), torch.zeros_like(dd))
            g = torch.where(m, g, torch.zeros_like(g))
            want += g @ ft[s0:s0 + 200_000]
        err = float(np.max(np.abs(qv[rows] - want.cpu().numpy())))
        bound = w["eps"] * float(np.abs(f0).sum())
        contract = {"targets": 1000, "max_abs_err": err, "bound_eps_sum_abs_f": bound, "ok": err <= bound}

    # batched right-hand sides (GMRES-style blocks, BASELINE config 5's "batch of
    # 8"): one apply of nrhs columns, D read once for all of them (k_spmm)
    batched = None
    if world == 1 and args.nrhs > 1 and R == 1:
        fb = np.stack([rhs(w, n, np.random.default_rng(SEED + 10 + r)) for r in range(args.nrhs)])
        fb_dev = torch.from_numpy(fb.view(np.float64).reshape(-1).copy()).cuda()
        qb_dev = torch.empty(2 * n * args.nrhs, dtype=torch.float64, device="cuda")

        def bstep():
            op.apply_device(fb_dev.data_ptr(), qb_dev.data_ptr(), args.nrhs, sh, f_is_real=f_real)
        bstep()
        torch.cuda.synchronize()
        op.set_profiling(True)
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 3
        b0.record(stream)
        for _ in range(reps):
            bstep()
        b1.record(stream)
        torch.cuda.synchronize()
        bst = op.stage_times()
        op.set_profiling(False)
        bms = b0.elapsed_time(b1) / reps
        spmv_ms = sum(ms for nm, ms in bst if nm == "spmv") / reps
        batched = {"nrhs": args.nrhs, "value": n * args.nrhs / (bms / 1e3), "unit": "points/s",
                   "ms_per_apply": round(bms, 3), "spmv_ms_per_apply": round(spmv_ms, 3),
                   "note": "one apply of nrhs right-hand sides; D' streamed once for up to 8 columns"}
        del fb_dev, qb_dev

    # the adjoint (conv_operator.cpp:311-324; GMRES / gradient callers): one
    # apply_adjoint per step on device buffers, 3 steps after a warm-up
    adjoint = None
    if world == 1 and R == 1 and args.adjoint:
        u_dev = torch.from_numpy((rng.standard_normal(n) + 1j * rng.standard_normal(n)).view(np.float64).copy()).cuda()
        p_dev = torch.empty(2 * n, dtype=torch.float64, device="cuda")
        op.apply_adjoint_device(u_dev.data_ptr(), p_dev.data_ptr(), 1, sh)
        torch.cuda.synchronize()
        op.set_profiling(True)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(3):
            op.apply_adjoint_device(u_dev.data_ptr(), p_dev.data_ptr(), 1, sh)
        a1.record(stream)
        torch.cuda.synchronize()
        ast = op.stage_times()
        op.set_profiling(False)
        ams = a0.elapsed_time(a1) / 3
        agg_a = {}
        for nm, ms in ast:
            agg_a[nm] = agg_a.get(nm, 0.0) + ms / 3
        adjoint = {"value": n / (ams / 1e3), "unit": "points/s", "ms_per_apply": round(ams, 3),
                   "stages_ms": {k: round(v, 3) for k, v in agg_a.items()},
                   "note": "apply_adjoint of a complex u on device buffers"}
        del u_dev, p_dev

    # procedural ring nodes (sbd_op_options.procedural_rings):
    # the same workload with the xi-side kernels regenerating every node and the
    # per-node arrays released -- apply time, HBM held, agreement with the
    # stored-array operator's q
    procedural = None
    if world == 1 and R == 1 and args.procedural:
        # (the operator goes through its file: a second GPU assembly beside the
        # resident operator would not fit its temporaries)
        ppath = f"/tmp/sbd_bench_proc_{os.getpid()}.sbdop"
        torch.cuda.empty_cache()  # the direct-sum check above leaves large cached blocks
        try:
            stored_bytes = int(info["device_bytes"])  # after assembly, before the adjoint's arrays were built
            op.save(ppath)
            pop = sbd.CompressedOperator.load(ppath, device=local, max_grid_bytes=96 << 30,
                                              options=sbd.OpOptions(procedural_rings=True))
            pinfo = pop.info()
            qp_dev = torch.empty(2 * n, dtype=torch.float64, device="cuda")
            for _ in range(3):
                pop.apply_device(f_dev.data_ptr(), qp_dev.data_ptr(), 1, sh, f_is_real=f_real)
            torch.cuda.synchronize()
            p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            p0.record(stream)
            for _ in range(5):
                pop.apply_device(f_dev.data_ptr(), qp_dev.data_ptr(), 1, sh, f_is_real=f_real)
            p1.record(stream)
            torch.cuda.synchronize()
            qp = qp_dev.view(-1, 2).cpu().numpy()
            qp = qp[:, 0] + 1j * qp[:, 1]
            procedural = {"on": bool(pinfo["procedural_rings"]),
                          "ms_per_apply": round(p0.elapsed_time(p1) / 5, 3),
                          "device_bytes": int(pinfo["device_bytes"]), "stored_device_bytes": stored_bytes,
                          "rel_l2_vs_stored": float(np.linalg.norm(qp - qv) / np.linalg.norm(qv)),
                          "note": "xi coordinates, phases and omega-hat regenerated in the kernels from (rho_p, "
                                  "M_p, weight_p, j); per-node arrays released; device_bytes of both operators "
                                  "before any adjoint"}
            del pop, qp_dev
        except Exception as exc:  # never fatal for the headline line
            procedural = {"error": str(exc)[:200]}
        finally:
            if os.path.exists(ppath):
                os.unlink(ppath)
        torch.cuda.empty_cache()

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if args.ref_full:
            parity, cpu = reference_same_config(op, f0, qv, 96 << 30)
        if cpu is None:
            kind, apply, fs, path = reference_sample(w, args.sample_n)
            per = min(time_reference(apply, fs, 1, 1) for _ in range(2))
            os.unlink(path)
            cpu = {"value": args.sample_n / per, "unit": "points/s", "cores": 1, "kind": kind,
                   "sample": (f"same distribution/eps/delta_min rule at N={args.sample_n}, "
                              "single-threaded CompressedOperator::apply, best of 2")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "points/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded clouds/RHS of the BASELINE.json shape)",
            "config": {"workload": w["desc"], "N": n, "nrhs": R, "n_xi": info["n_xi"], "nnz": info["nnz"],
                       "P": info["P"], "w": info["w"], "grid": [info["n1_in"], info["n2_in"]],
                       "nufft_tol": info["nufft_tol"],
                       "l2": "inputs larger than L2 (grid + xi + D >> 126 MB)",
                       "parallelism": "single" if world == 1 else
                       ((f"slab x{world}: grids, xi nodes and targets split by position, two all-to-alls"
                         if scheme == "slab" else
                         f"sharded x{world}: sources/targets/D rows split, all-reduce of the xi spectrum") +
                        (f" (gloo; {world} ranks share {ndev} GPU(s): functional run, not a scaling number)"
                         if shared else " (NCCL)")),
                       "offline_s": round(t_offline, 2)},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": n * R / e2e_s, "unit": "points/s",
                    "h2d_bytes_per_step": 16 * n * R, "d2h_bytes_per_step": 16 * n * R},
            "e2e_pipelined": e2e_pipe,
            "gpu_launches": launches,
            "clocks": clk,
            "batched_rhs": batched,
            "adjoint": adjoint,
            "procedural_rings": procedural,
            "rhs_parallel": rhs_par,
            "other_scheme": alt,
            "contract": contract,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="4")
    ap.add_argument("--scale", type=float, default=1.0, help="multiply the config's N (testing)")
    ap.add_argument("--sample-n", type=int, default=50000, help="reference CPU sample size")
    ap.add_argument("--ref-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nrhs", type=int, default=8, help="also time one batched apply of this many RHS (1: off)")
    ap.add_argument("--adjoint", type=int, default=1, help="1: also time apply_adjoint")
    ap.add_argument("--procedural", type=int, default=1,
                    help="1: also time the apply with procedural ring nodes (a second assemble)")
    ap.add_argument("--scheme", default="auto", choices=["auto", "slab", "shard"],
                    help="multi-GPU apply for N > 1: slab decomposition or the north_star source/target sharding")
    ap.add_argument("--ref-full", type=int, default=1,
                    help="1: one reference apply of the full config on one core after the timed region "
                         "(parity + same-config cpu_baseline; ~5 min at config 4); 0: the N=5e4 sample only")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(spawn_ranks(args))
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    w = workload(args.config, args.scale)
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_b200(args, w)


if __name__ == "__main__":
    main()
