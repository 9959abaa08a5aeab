"""GPU: the sharded apply's device halves (sbd_op_forward_spectrum /
sbd_op_backward_targets) with G shards emulated on one B200 -- the
all-reduce is a plain sum here (the collective itself is covered over gloo in
tests/test_parallel.py; nothing in this run has more than one GPU)."""
import numpy as np
import pytest
import torch

import paper_1711_07877_b200 as sbd
from paper_1711_07877_b200.parallel import DeviceBackend, ShardedApply
from tests.conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["lap_disk_n1000", "helm_disk_n800", "lap_two_clouds",
                                  "lap_star_n1500"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_halves_reproduce_apply(name, world):
    path, g = golden(name)
    # the full-path operator (every xi node) and the default one (the
    # real-input half split for a real f) are sharded alike; each must
    # reproduce its own single-device apply
    op_full = sbd.CompressedOperator.load(path, options=sbd.OpOptions(real_input_split=False))
    op_default = sbd.CompressedOperator.load(path)
    f = torch.from_numpy(np.ascontiguousarray(g["f"], dtype=np.complex128).view(np.float64)).cuda()
    for op in (op_full, op_default):
        be = DeviceBackend(op)
        ranks = [ShardedApply(be, r, world, allreduce=lambda t: None) for r in range(world)]
        n = be.spectrum_length(f)
        total = be.new_spectrum()
        for r, sa in enumerate(ranks):
            spec = be.new_spectrum()
            be.forward_spectrum(f, sa.src[r], sa.src[r + 1], spec)
            total[: 2 * n] += spec[: 2 * n]
        q = torch.zeros(2 * be.n_tgt, dtype=torch.float64, device="cuda")
        for r, sa in enumerate(ranks):
            be.backward_targets(total, f, sa.tgt[r], sa.tgt[r + 1], q)
        torch.cuda.synchronize()
        qh = q.cpu().numpy().view(np.complex128)
        assert rel_l2(qh, op.apply(g["f"])) <= 1e-13
        assert rel_l2(qh, g["q"]) <= 1e-9


@pytest.mark.parametrize("name", ["lap_disk_n1000", "helm_disk_n800"])
def test_sharded_halves_on_procedural_operator(name):
    # the sharded halves run the same xi-side kernels: with procedural ring
    # nodes they regenerate the nodes of their output / point ranges from the ids
    path, g = golden(name)
    op = sbd.CompressedOperator.load(path, options=sbd.OpOptions(procedural_rings=True))
    assert op.info()["procedural_rings"] == 1
    f = torch.from_numpy(np.ascontiguousarray(g["f"], dtype=np.complex128).view(np.float64)).cuda()
    be = DeviceBackend(op)
    world = 3
    ranks = [ShardedApply(be, r, world, allreduce=lambda t: None) for r in range(world)]
    n = be.spectrum_length(f)
    total = be.new_spectrum()
    for r, sa in enumerate(ranks):
        spec = be.new_spectrum()
        be.forward_spectrum(f, sa.src[r], sa.src[r + 1], spec)
        total[: 2 * n] += spec[: 2 * n]
    q = torch.zeros(2 * be.n_tgt, dtype=torch.float64, device="cuda")
    for r, sa in enumerate(ranks):
        be.backward_targets(total, f, sa.tgt[r], sa.tgt[r + 1], q)
    torch.cuda.synchronize()
    qh = q.cpu().numpy().view(np.complex128)
    assert rel_l2(qh, op.apply(g["f"])) <= 1e-13
    assert rel_l2(qh, g["q"]) <= 1e-9
