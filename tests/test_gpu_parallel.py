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
def test_sharded_halves_reproduce_apply(name, world, monkeypatch):
    path, g = golden(name)
    # the sharded halves compute every xi node: compare with the full-path
    # operator bitwise-closely, and with the default one (which may take the
    # real-input half split) to the half split's own agreement
    monkeypatch.setenv("SBD_NO_HERM", "1")
    op = sbd.CompressedOperator.load(path)
    monkeypatch.delenv("SBD_NO_HERM")
    op_default = sbd.CompressedOperator.load(path)
    be = DeviceBackend(op)
    f = torch.from_numpy(np.ascontiguousarray(g["f"], dtype=np.complex128).view(np.float64)).cuda()
    ranks = [ShardedApply(be, r, world, allreduce=lambda t: None) for r in range(world)]
    total = be.new_spectrum()
    for r, sa in enumerate(ranks):
        spec = be.new_spectrum()
        be.forward_spectrum(f, sa.src[r], sa.src[r + 1], spec)
        total += spec
    q = torch.zeros(2 * be.n_tgt, dtype=torch.float64, device="cuda")
    for r, sa in enumerate(ranks):
        be.backward_targets(total, f, sa.tgt[r], sa.tgt[r + 1], q)
    torch.cuda.synchronize()
    qh = q.cpu().numpy().view(np.complex128)
    assert rel_l2(qh, op.apply(g["f"])) <= 1e-13
    qd = op_default.apply(g["f"])
    assert rel_l2(qh.real, qd.real) <= 1e-13 and rel_l2(qh, qd) <= 5e-10
    assert rel_l2(qh, g["q"]) <= 1e-9
