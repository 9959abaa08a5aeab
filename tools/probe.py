"""Dev probe (not part of the product): build a reference operator at size N
with the compiled reference (oracle/_ref), load it on the GPU, check parity
against the C oracle and print per-stage CUDA-event times."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1711_07877_b200 as sbd  # noqa: E402
from oracle.oracle import Oracle, RefLib  # noqa: E402
from tests.clouds import disk_cloud  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
path = f"/tmp/probe_{N}.sbdop"
rng = np.random.default_rng(7)
z = disk_cloud(N, rng)
ref = RefLib()
t0 = time.time()
if not os.path.exists(path):
    d = ref.diameter(z)
    info = ref.assemble_save(path, z, a_override=(2.74 / np.sqrt(N)) / d, eps=1e-6,
                             max_grid_bytes=16 << 30)
    print("ref assemble", time.time() - t0, info, flush=True)
t0 = time.time()
op = sbd.CompressedOperator.load(path, max_grid_bytes=16 << 30)
print("gpu load", time.time() - t0, op.info(), flush=True)
f = rng.standard_normal(N) + 0j
q = op.apply(f)
t0 = time.time()
qo = Oracle().op(path, max_grid_bytes=16 << 30).apply(f)
print("oracle apply s", time.time() - t0)
print("rel_l2 vs oracle", np.linalg.norm(q - qo) / np.linalg.norm(qo), flush=True)
op.set_profiling(True)
for it in range(3):
    op.apply(f)
    st = op.stage_times()
    print(" ".join(f"{n}={ms:.3f}" for n, ms in st), "total", sum(ms for _, ms in st))
import torch  # noqa: E402
fd = torch.tensor(np.ascontiguousarray(f).view(np.float64), device="cuda")
qd = torch.empty(2 * N, dtype=torch.float64, device="cuda")
op.set_profiling(False)
for _ in range(3):
    op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    op.apply_device(fd.data_ptr(), qd.data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"apply device {ms:.3f} ms -> {N / ms * 1e3:.3e} points/s")
