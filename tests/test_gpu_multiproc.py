"""GPU, two processes: the sharded apply (paper_1711_07877_b200/parallel.py)
through torch.distributed with real ranks -- DeviceBackend on the device,
the xi-spectrum all-reduce as an actual collective (gloo over CUDA tensors:
this box has one GPU, NCCL refuses two ranks on one device) -- against the
reference golden. The two ranks only meet in the host-mediated collective;
no kernel waits on another rank's kernel. The same script is what
`bench.py --gpus N` runs per rank."""
import os
import sys

import numpy as np
import pytest

from tests.conftest import ROOT, golden, rel_l2

pytestmark = pytest.mark.gpu


def _rank(rank, world, init, names, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    import paper_1711_07877_b200 as sbd
    from paper_1711_07877_b200.parallel import DeviceBackend, ShardedApply

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=init, rank=rank, world_size=world)
    for name in names:
        path, g = golden(name)
        op = sbd.CompressedOperator.load(path)
        for label, f in (("golden", g["f"]),
                         ("real", np.random.default_rng(3).standard_normal(len(g["f"])) + 0j)):
            fd = torch.from_numpy(np.ascontiguousarray(f, dtype=np.complex128).view(np.float64).copy()).cuda()
            sa = ShardedApply(DeviceBackend(op), rank, world)
            q = torch.zeros(2 * op.n_tgt(), dtype=torch.float64, device="cuda")
            sa.apply(fd, q)
            torch.cuda.synchronize()
            dist.all_reduce(q)  # every rank wrote only its target shard
            if rank == 0:
                np.save(os.path.join(out_dir, f"{name}_{label}.npy"), q.cpu().numpy().view(np.complex128))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_sharded_apply_matches_golden(tmp_path):
    import torch.multiprocessing as mp
    names = ["lap_disk_n1000", "helm_disk_n800", "lap_two_clouds"]
    init = "file://" + str(tmp_path / "store")
    mp.spawn(_rank, args=(2, init, names, str(tmp_path)), nprocs=2, join=True)
    import paper_1711_07877_b200 as sbd
    for name in names:
        path, g = golden(name)
        assert rel_l2(np.load(tmp_path / f"{name}_golden.npy"), g["q"]) <= 1e-9, name
        f = np.random.default_rng(3).standard_normal(len(g["f"])) + 0j
        want = sbd.CompressedOperator.load(path).apply(f)
        assert rel_l2(np.load(tmp_path / f"{name}_real.npy"), want) <= 1e-13, name


def test_bench_gpus_2_runs_two_ranks():
    # `bench.py --gpus N` must start N ranks itself (re-exec under
    # torch.distributed.run) and report n_gpus = N; on this one-GPU box the two
    # ranks share the device over gloo (a functional run, labelled as such)
    import json
    import subprocess
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "1",
                        "--steps", "3", "--warmup", "3", "--nrhs", "1", "--no-cpu-baseline"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2
    assert line["contract"]["ok"]
    # both partitions are timed; the headline is the faster one (--scheme auto)
    par, other = line["config"]["parallelism"], line["other_scheme"]
    assert ("slab x2" in par and other["scheme"] == "shard") or ("sharded x2" in par and other["scheme"] == "slab")
    assert line["value"] >= other["value"]
    assert line["rhs_parallel"]["scaling"] == "weak"
    forced = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "1",
                             "--steps", "2", "--warmup", "3", "--nrhs", "1", "--no-cpu-baseline", "--scheme", "slab",
                             "--adjoint", "0", "--procedural", "0"],
                            capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert forced.returncode == 0, forced.stderr[-3000:]
    fl = json.loads([x for x in forced.stdout.splitlines() if x.startswith("{")][-1])
    assert "slab x2" in fl["config"]["parallelism"] and fl["contract"]["ok"]
