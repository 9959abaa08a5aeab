"""The multi-GPU orchestration (paper_1711_07877_b200/parallel.py) on CPU:
world_size 2 over gloo, with the C oracle as each rank's compute backend
(test-only), checked against the reference's golden apply output. The same
ShardedApply drives sbd_op_forward_spectrum / sbd_op_backward_targets on the
GPU (tests/test_gpu_parallel.py emulates the shards on one device)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.conftest import golden, rel_l2


class OracleBackend:
    """Per-rank compute on the CPU oracle; 'sorted order' = caller order."""

    def __init__(self, path):
        from oracle.oracle import Oracle
        self.op = Oracle().op(path)
        self.w = self.op.weights()
        self.n_src, self.n_tgt, self.n_xi = self.op.n_src, self.op.n_tgt, self.op.n_xi

    def shard_bounds(self, side, nshards):
        n = self.n_src if side == 0 else self.n_tgt
        return [n * i // nshards for i in range(nshards + 1)]

    def new_spectrum(self):
        return torch.zeros(2 * self.n_xi, dtype=torch.float64)

    def forward_spectrum(self, f, lo, hi, spec):
        fc = f.numpy().view(np.complex128).copy()
        fc[:lo] = 0
        fc[hi:] = 0
        spec.copy_(torch.from_numpy(self.op.stage(1, fc).view(np.float64)))

    def backward_targets(self, spec, f, lo, hi, q):
        s = spec.numpy().view(np.complex128) * self.w
        full = self.op.stage(2, s)
        full = self.op.stage(3, f.numpy().view(np.complex128), out=full)
        q.numpy().view(np.complex128)[lo:hi] = full[lo:hi]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_07877_b200.parallel import ShardedApply
    path, g = golden(name)
    be = OracleBackend(path)
    sa = ShardedApply(be, rank, world)
    f = torch.from_numpy(np.ascontiguousarray(g["f"], dtype=np.complex128).view(np.float64))
    q = torch.zeros(2 * be.n_tgt, dtype=torch.float64)
    lo, hi = sa.apply(f, q)
    # gather the target shards (disjoint, zeros elsewhere) for the check
    dist.all_reduce(q)
    if rank == 0:
        np.save(os.path.join(outdir, "q.npy"), q.numpy().view(np.complex128))
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["lap_disk_n1000", "helm_disk_n800", "lap_two_clouds"])
def test_sharded_apply_gloo_world2(name, tmp_path):
    mp.spawn(_worker, args=(2, _free_port(), name, str(tmp_path)), nprocs=2, join=True)
    q = np.load(tmp_path / "q.npy")
    _, g = golden(name)
    assert rel_l2(q, g["q"]) <= 1e-12


def test_shard_bounds_partition():
    from paper_1711_07877_b200.parallel import ShardedApply

    class Dummy(OracleBackend):
        def __init__(self):
            self.n_src, self.n_tgt, self.n_xi = 10, 7, 3

    for world in (1, 2, 3, 8):
        sa = ShardedApply(Dummy(), 0, world, allreduce=lambda t: None)
        assert sa.src[0] == 0 and sa.src[-1] == 10 and sa.tgt[-1] == 7
        assert all(a <= b for a, b in zip(sa.src, sa.src[1:]))


def _a2a_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1711_07877_b200.parallel import dist_alltoall
    # rank r sends (r + 1) * (k + 1) values "r.k" to rank k, back to back
    ssp = [(rank + 1) * (k + 1) for k in range(world)]
    send = torch.cat([torch.full((n,), 10.0 * rank + k, dtype=torch.float64) for k, n in enumerate(ssp)])
    rsp = [(k + 1) * (rank + 1) for k in range(world)]
    recv = torch.zeros(sum(rsp) + 3, dtype=torch.float64)  # (oversized, as SlabApply allocates)
    dist_alltoall(recv, send, rsp, ssp)
    np.save(os.path.join(outdir, f"a2a_{rank}.npy"), recv.numpy())
    dist.destroy_process_group()


def test_slab_exchange_over_gloo(tmp_path):
    # the slab decomposition's two all-to-alls (parallel.dist_alltoall) route
    # each rank's block for rank k to rank k, in rank order
    world = 2
    mp.spawn(_a2a_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        got = np.load(tmp_path / f"a2a_{r}.npy")
        want = np.concatenate([np.full((k + 1) * (r + 1), 10.0 * k + r) for k in range(world)])
        assert np.array_equal(got[:len(want)], want)
