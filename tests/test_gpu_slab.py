"""GPU: the slab decomposition (csrc/slab.cpp) with G
ranks emulated on one B200 -- every rank's stages run in turn and the two
all-to-alls are device copies between the ranks' buffers (nothing in this run
has more than one GPU; the NCCL/gloo exchange itself is
paper_1711_07877_b200.parallel.dist_alltoall, covered over gloo on CPU and
by the two-process test below). The assembled q must equal the single-device
apply of the complex pipeline to rounding and the reference golden to 1e-9:
no stage is replicated, every partition is exercised (1, 2, 3, 8 ranks).
Rounding differs from the single-device pipeline (plain transforms instead
of the radix-folded ones, other summation orders): 1e-11 relative."""
import os
import sys

import numpy as np
import pytest
import torch

import paper_1711_07877_b200 as sbd
from paper_1711_07877_b200.parallel import SlabApply
from tests.conftest import ROOT, golden, rel_l2

pytestmark = pytest.mark.gpu

NAMES = ["lap_disk_n1000", "helm_disk_n800", "lap_two_clouds", "lap_star_n1500"]


def emulated_apply(op, f_np, world):
    f = torch.from_numpy(np.ascontiguousarray(f_np, dtype=np.complex128).view(np.float64).copy()).cuda()
    q = torch.zeros(2 * op.n_tgt(), dtype=torch.float64, device="cuda")
    ranks = [SlabApply(op, r, world, alltoall=lambda *a: None) for r in range(world)]

    def exchange(e):
        # rank r's receive block from rank k = rank k's send block for r
        for r, dst in enumerate(ranks):
            recv = dst.bufs[e][1]
            ro = 0
            for k, src in enumerate(ranks):
                ssp = src.splits[e][0]
                so = sum(ssp[:r])
                n = ssp[r]
                assert n == dst.splits[e][1][k]
                recv[ro:ro + n].copy_(src.bufs[e][0][so:so + n])
                ro += n

    for s in ranks:
        s.stage(0, None, f, s.bufs[0][0])
    exchange(0)
    for s in ranks:
        s.stage(1, s.bufs[0][1], None, s.bufs[1][0])
    exchange(1)
    for s in ranks:
        s.stage(2, s.bufs[1][1], f, q)
    torch.cuda.synchronize()
    return q.cpu().numpy().view(np.complex128)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_slab_emulated_matches_apply(name, world):
    path, g = golden(name)
    op = sbd.CompressedOperator.load(path, options=sbd.OpOptions(real_input_split=False))
    full = op.apply(g["f"])
    q = emulated_apply(op, g["f"], world)
    assert rel_l2(q, full) <= 1e-11
    assert rel_l2(q, g["q"]) <= 1e-9
    fc = np.random.default_rng(7).standard_normal(len(g["f"])) + 1j * np.random.default_rng(8).standard_normal(len(g["f"]))
    assert rel_l2(emulated_apply(op, fc, world), op.apply(fc)) <= 1e-11


def test_slab_on_procedural_operator():
    # an operator loaded with procedural ring nodes has released its per-node
    # arrays; creating the slab plan rebuilds them (same device functions), and
    # the forward apply keeps regenerating the nodes in its kernels
    path, g = golden("lap_star_n1500")
    op = sbd.CompressedOperator.load(path, options=sbd.OpOptions(real_input_split=False, procedural_rings=True))
    assert op.info()["procedural_rings"] == 1
    q = emulated_apply(op, g["f"], 3)
    assert rel_l2(q, g["q"]) <= 1e-9
    assert rel_l2(op.apply(g["f"]), g["q"]) <= 1e-9


def test_slab_emulated_at_scale():
    # the config-4 distribution at N = 2e5 (grid > 4096, radix passes in the
    # single-device pipeline; the slab path runs plain transforms)
    from tests.clouds import disk_cloud
    n = 200_000
    z = disk_cloud(n, np.random.default_rng(909))
    dmax = sbd.cloud_diameter(z)
    op = sbd.CompressedOperator.assemble(
        sbd.kernel_laplace(), z,
        opts=sbd.AssembleOptions(eps=1e-6, a_override=(2.74 / np.sqrt(n)) / dmax,
                                 pipeline=sbd.OpOptions(real_input_split=False)))
    f = np.random.default_rng(910).standard_normal(n) + 0j
    want = op.apply(f)
    for world in (2, 8):
        assert rel_l2(emulated_apply(op, f, world), want) <= 1e-11, world


def _rank(rank, world, init, name, out):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=init, rank=rank, world_size=world)
    path, g = golden(name)
    op = sbd.CompressedOperator.load(path, options=sbd.OpOptions(real_input_split=False))
    sa = SlabApply(op, rank, world)  # default exchange: parallel.dist_alltoall
    f = torch.from_numpy(np.ascontiguousarray(g["f"], dtype=np.complex128).view(np.float64).copy()).cuda()
    q = torch.zeros(2 * op.n_tgt(), dtype=torch.float64, device="cuda")
    sa.apply(f, q)
    torch.cuda.synchronize()
    dist.all_reduce(q)  # every rank wrote only its own targets
    if rank == 0:
        np.save(out, q.cpu().numpy().view(np.complex128))
    dist.barrier()
    dist.destroy_process_group()


def test_slab_two_processes(tmp_path):
    import torch.multiprocessing as mp
    name = "helm_disk_n800"
    out = str(tmp_path / "q.npy")
    mp.spawn(_rank, args=(2, "file://" + str(tmp_path / "store"), name, out), nprocs=2, join=True)
    path, g = golden(name)
    assert rel_l2(np.load(out), g["q"]) <= 1e-9
