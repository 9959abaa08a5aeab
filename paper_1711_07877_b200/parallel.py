"""Multi-GPU apply: one process per GPU, torch.distributed for the plumbing.

The north_star partition of CompressedOperator::apply (conv_operator.cpp:301-309)
over G ranks:

  1. sources sharded: rank r forms the omega-hat-weighted xi spectrum of its
     source shard only (sbd_op_forward_spectrum); the spectrum is linear in f,
  2. one all-reduce (sum) of the n_xi complex spectrum -- the only data-path
     collective, because it is the path's only real exchange step (for a
     real f on a half-split operator only the computed half: n_xi / 2),
  3. targets and near-field rows sharded: rank r evaluates the second NUFFT at
     its target shard and adds its rows of D f (sbd_op_backward_targets); f is
     replicated (all-gathered) on every rank.

Shards are ranges of the operator's spatially sorted orders, so a rank's
points are spatially compact. The orchestration is backend-agnostic: the GPU
backend calls the C ABI on device buffers; tests drive the same code with a
CPU backend over gloo.
"""
from __future__ import annotations

import ctypes

from ._capi import check, lib


class DeviceBackend:
    """CompressedOperator on this rank's GPU, torch tensors as buffers."""

    def __init__(self, op):
        import torch
        self.torch = torch
        self.op = op
        info = op.info()
        self.n_src, self.n_tgt, self.n_xi = info["n_src"], info["n_tgt"], info["n_xi"]
        if not (info["fast_in"] and info["fast_out"]):
            raise ValueError("sharded apply needs both NUFFTs on the gridded path")

    def shard_bounds(self, side: int, nshards: int):
        b = (ctypes.c_uint64 * (nshards + 1))()
        check(lib.sbd_op_shard_bounds(self.op._h, side, nshards, b))
        return [int(x) for x in b]

    def new_spectrum(self):
        return self.torch.zeros(2 * self.n_xi, dtype=self.torch.float64, device="cuda")

    def forward_spectrum(self, f, lo, hi, spec):
        s = self.torch.cuda.current_stream().cuda_stream
        check(lib.sbd_op_forward_spectrum(self.op._h, ctypes.c_void_p(f.data_ptr()), lo, hi,
                                          ctypes.c_void_p(spec.data_ptr()), ctypes.c_void_p(s)))

    def spectrum_length(self, f):
        """Leading spectrum entries formed / reduced / read for this f
        (sbd_op_spectrum_length: the computed half for a real f)."""
        n = ctypes.c_uint64()
        s = self.torch.cuda.current_stream().cuda_stream
        check(lib.sbd_op_spectrum_length(self.op._h, ctypes.c_void_p(f.data_ptr()), ctypes.c_void_p(s),
                                         ctypes.byref(n)))
        return int(n.value)

    def backward_targets(self, spec, f, lo, hi, q):
        s = self.torch.cuda.current_stream().cuda_stream
        check(lib.sbd_op_backward_targets(self.op._h, ctypes.c_void_p(spec.data_ptr()),
                                          ctypes.c_void_p(f.data_ptr()), lo, hi,
                                          ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(s)))


class ShardedApply:
    """q = A f split over `world` ranks (see module docstring).

    `f` (2 * n_src float64, interleaved complex) is replicated on every rank;
    each rank's `q` receives the entries of its target shard (at their caller
    indices) and is left untouched elsewhere."""

    def __init__(self, backend, rank: int, world: int, allreduce=None):
        self.b = backend
        self.rank, self.world = rank, world
        self.src = backend.shard_bounds(0, world)
        self.tgt = backend.shard_bounds(1, world)
        if allreduce is None:
            import torch.distributed as dist
            allreduce = (lambda t: dist.all_reduce(t)) if world > 1 else (lambda t: None)
        self.allreduce = allreduce
        self.spec = backend.new_spectrum()

    def target_range(self):
        return self.tgt[self.rank], self.tgt[self.rank + 1]

    def apply(self, f, q):
        r = self.rank
        # a real f on a half-split operator only forms (and reduces) the
        # computed half of the spectrum
        n = self.b.spectrum_length(f) if hasattr(self.b, "spectrum_length") else self.b.n_xi
        self.b.forward_spectrum(f, self.src[r], self.src[r + 1], self.spec)
        self.allreduce(self.spec[: 2 * n])
        self.b.backward_targets(self.spec, f, self.tgt[r], self.tgt[r + 1], q)
        return self.target_range()


def dist_alltoall(recv, send, recv_splits, send_splits):
    """The slab exchanges over torch.distributed: NCCL moves device buffers
    directly; gloo (CPU tests, ranks sharing one GPU) goes through host copies."""
    import torch.distributed as dist
    n_r, n_s = sum(recv_splits), sum(send_splits)
    if dist.get_backend() == "nccl" or not send.is_cuda:
        dist.all_to_all_single(recv[:n_r], send[:n_s], recv_splits, send_splits)
        return
    r = recv[:n_r].cpu()
    dist.all_to_all_single(r, send[:n_s].cpu(), recv_splits, send_splits)
    recv[:n_r].copy_(r)


class SlabApply:
    """q = A f over `world` ranks with no replicated stage: the slab
    decomposition of csrc/slab.cpp. Each rank holds the
    operator; `alltoall(recv, send, recv_splits, send_splits)` moves the two
    exchanges (torch.distributed.all_to_all_single over NCCL by default; the
    single-GPU emulation in tests/ passes its own). `f` (2 n_src float64,
    interleaved complex, device) is replicated; `q` receives this rank's
    targets at their caller indices."""

    def __init__(self, op, rank: int, world: int, alltoall=None):
        import torch
        self.torch = torch
        self.op, self.rank, self.world = op, rank, world
        h = ctypes.c_void_p()
        check(lib.sbd_slab_create(op._h, rank, world, ctypes.byref(h)))
        self._h = h
        self.splits = []
        for e in (0, 1):
            snd = (ctypes.c_uint64 * world)()
            rcv = (ctypes.c_uint64 * world)()
            check(lib.sbd_slab_counts(h, e, snd, rcv))
            self.splits.append(([2 * int(x) for x in snd], [2 * int(x) for x in rcv]))
        self.bufs = [(torch.empty(max(sum(s), 2), dtype=torch.float64, device="cuda"),
                      torch.empty(max(sum(r), 2), dtype=torch.float64, device="cuda")) for s, r in self.splits]
        self.alltoall = alltoall or dist_alltoall

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:
            try:
                lib.sbd_slab_destroy(self._h)
            except Exception:  # interpreter shutdown
                pass
            self._h = None

    def stage(self, k, d_in, d_f, d_out):
        s = self.torch.cuda.current_stream().cuda_stream
        ptr = lambda t: None if t is None else ctypes.c_void_p(t.data_ptr())  # noqa: E731
        check(lib.sbd_slab_stage(self._h, k, ptr(d_in), ptr(d_f), ptr(d_out), ctypes.c_void_p(s)))

    def exchange(self, e):
        send, recv = self.bufs[e]
        ssp, rsp = self.splits[e]
        self.alltoall(recv, send, rsp, ssp)

    def apply(self, f, q):
        self.stage(0, None, f, self.bufs[0][0])
        self.exchange(0)
        self.stage(1, self.bufs[0][1], None, self.bufs[1][0])
        self.exchange(1)
        self.stage(2, self.bufs[1][1], f, q)
