"""Python mirror of the reference operator API, over the C ABI.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/sbd/conv_operator.hpp, nufft.hpp, kernels.hpp,
point_cloud.hpp) so that tests read like the reference's own tests:

  reference (C++)                              here
  -------------------------------------------  ------------------------------------------
  kernel_laplace() / kernel_helmholtz(k)       kernel_laplace() / kernel_helmholtz(k)
  make_cloud(std::vector<Vec2>)                make_cloud(points (n,2))
  AssembleOptions{eps, alpha, a_override, ..}  AssembleOptions(eps=..., ...)
  CompressedOperator::assemble(kernel, s[, t], opts) CompressedOperator.assemble(...)
  CompressedOperator::load(path) / save(path)  CompressedOperator.load(path) / .save(path)
  op.apply(f) -> std::vector<cplx>             op.apply(f) -> np.ndarray[complex128]
  op.apply_adjoint(u)                          op.apply_adjoint(u)
  NufftPlan(points, freqs, sign, opts)         NufftPlan(points, freqs, sign, NufftOptions())
  ndft_direct(points, freqs, coeffs, sign)     ndft_direct(points, freqs, coeffs, sign)
  std::invalid_argument / domain_error / runtime_error -> ValueError / DomainError / SbdError

Everything computes on the GPU through libsbd_b200.so; there is no CPU path.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import numpy as np

from . import _capi
from ._capi import check, lib

_dp = ctypes.POINTER(ctypes.c_double)


def _xy(points) -> np.ndarray:
    a = np.ascontiguousarray(points, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(-1, 2)
    if a.ndim != 2 or a.shape[1] != 2:
        raise ValueError("points must have shape (n, 2)")
    return a


def _cx(v) -> np.ndarray:
    return np.ascontiguousarray(v, dtype=np.complex128)


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


# --------------------------------------------------------------- kernels
@dataclasses.dataclass(frozen=True)
class KernelSpec:
    """kernels.hpp:59-68. kind 'laplace' (G = log r) or 'helmholtz'
    (G = -(i/4) H0^(1)(k r) = Y0(kr)/4 - i J0(kr)/4)."""
    kind: str = "laplace"
    k: float = 0.0

    @property
    def code(self) -> int:
        return {"laplace": 0, "helmholtz": 1}[self.kind]

    def is_complex(self) -> bool:
        return self.kind == "helmholtz"


def kernel_laplace() -> KernelSpec:
    return KernelSpec("laplace", 0.0)


def kernel_helmholtz(k: float) -> KernelSpec:
    if not k > 0.0:
        raise _capi.DomainError("kernel_helmholtz: k must be positive")
    return KernelSpec("helmholtz", float(k))


@dataclasses.dataclass
class PointCloud:
    points: np.ndarray
    diameter: float = 0.0

    def size(self) -> int:
        return len(self.points)


def cloud_diameter(points) -> float:
    """Exact diameter (convex hull + rotating calipers, point_cloud.cpp:39-57)."""
    p = _xy(points)
    return float(lib.sbd_cloud_diameter(_ptr(p), len(p)))


def make_cloud(points) -> PointCloud:
    """point_cloud.hpp:20."""
    p = _xy(points)
    return PointCloud(p, cloud_diameter(p))


@dataclasses.dataclass
class OpOptions:
    """sbd_op_options (include/sbd_b200.h): the pipeline choices of one
    operator. Every combination computes the same operator within the parity
    bar; the defaults are the fastest path."""
    real_input_split: bool = True
    hermitian_fft: bool = True
    radix_first_pass: int = -1   # -1 auto, 0 off, 1 force
    spread_kernel: str = "lists"  # lists | bins | warp | scalar
    interp_kernel: str = "auto"   # auto | tile | mma | scalar
    fused: bool = True
    verbose: bool = False
    procedural_rings: bool = False  # regenerate the xi nodes in the kernels instead of storing their arrays

    def _c(self) -> _capi.OpOptionsC:
        sk = {"lists": 0, "bins": 1, "warp": 2, "scalar": 3}[self.spread_kernel]
        ik = {"auto": 0, "tile": 1, "mma": 2, "scalar": 3}[self.interp_kernel]
        return _capi.OpOptionsC(int(self.real_input_split), int(self.hermitian_fft),
                                int(self.radix_first_pass), sk, ik, int(self.fused), int(self.verbose),
                                int(self.procedural_rings))


@dataclasses.dataclass
class AssembleOptions:
    """conv_operator.hpp:24-31 plus the CUDA device ordinal and the pipeline
    options."""
    eps: float = 1e-6
    alpha: float = 0.0
    a_override: float = 0.0
    small_k_factor: float = 0.5
    nufft_direct_threshold: int = 1 << 20
    max_grid_bytes: int = 4 << 30
    device: int = 0
    pipeline: OpOptions = dataclasses.field(default_factory=OpOptions)

    def _c(self) -> _capi.AssembleOptionsC:
        return _capi.AssembleOptionsC(self.eps, self.alpha, self.a_override, self.small_k_factor,
                                      self.nufft_direct_threshold, self.max_grid_bytes,
                                      self.device, self.pipeline._c())


@dataclasses.dataclass
class FrequencyQuadrature:
    freqs: np.ndarray
    weights: np.ndarray
    ring_offsets: np.ndarray

    def size(self) -> int:
        return len(self.freqs)


@dataclasses.dataclass
class SparsePairMatrix:
    row_offsets: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    def nnz(self) -> int:
        return len(self.values)


def choose_parameters(n: int, eps: float, alpha: float):
    """conv_operator.cpp:121-133 -> (a, P_hint)."""
    a = ctypes.c_double()
    p = ctypes.c_int()
    check(lib.sbd_choose_parameters(int(n), float(eps), float(alpha), ctypes.byref(a),
                                    ctypes.byref(p)))
    return a.value, p.value


# --------------------------------------------------------------- operator
class CompressedOperator:
    """conv_operator.hpp:37-79 on one B200."""

    def __init__(self, handle: ctypes.c_void_p):
        self._h = handle
        self._info = None

    # -- construction
    @staticmethod
    def assemble(kernel: KernelSpec, source, target=None,
                 opts: Optional[AssembleOptions] = None) -> "CompressedOperator":
        opts = opts or AssembleOptions()
        s = _xy(source.points if isinstance(source, PointCloud) else source)
        t = None
        if target is not None:
            t = _xy(target.points if isinstance(target, PointCloud) else target)
            if t.shape == s.shape and np.array_equal(t, s):
                t = None  # conv_operator.cpp:252: identical clouds -> single-cloud operator
        h = ctypes.c_void_p()
        oc = opts._c()
        check(lib.sbd_op_assemble(kernel.code, kernel.k, _ptr(s), len(s), _ptr(t),
                                  0 if t is None else len(t), ctypes.byref(oc), ctypes.byref(h)))
        return CompressedOperator(h)

    @staticmethod
    def load(path: str, device: int = 0, max_grid_bytes: int = 0,
             options: Optional[OpOptions] = None) -> "CompressedOperator":
        """conv_operator.cpp:449-490 (max_grid_bytes 0 = the reference's 4 GiB)."""
        h = ctypes.c_void_p()
        oc = (options or OpOptions())._c()
        check(lib.sbd_op_load_ex(str(path).encode(), int(device), int(max_grid_bytes),
                                 ctypes.byref(oc), ctypes.byref(h)))
        return CompressedOperator(h)

    def save(self, path: str) -> None:
        check(lib.sbd_op_save(self._h, str(path).encode()))

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.sbd_op_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- info / accessors
    def info(self) -> dict:
        i = _capi.OpInfoC()
        check(lib.sbd_op_info(self._h, ctypes.byref(i)))
        return {f: getattr(i, f) for f, _ in _capi.OpInfoC._fields_}

    def _get(self, which, dtype, shape_tail=()):
        n = ctypes.c_uint64()
        check(lib.sbd_op_get(self._h, which, None, ctypes.byref(n)))
        a = np.empty(n.value, dtype=dtype)
        check(lib.sbd_op_get(self._h, which, a.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n)))
        return a

    def n_src(self) -> int:
        return int(self.info()["n_src"])

    def n_tgt(self) -> int:
        return int(self.info()["n_tgt"])

    def source(self) -> PointCloud:
        return PointCloud(self._get(0, np.float64).reshape(-1, 2))

    def target(self) -> PointCloud:
        return PointCloud(self._get(1, np.float64).reshape(-1, 2))

    def single_cloud(self) -> bool:
        return bool(self.info()["single_cloud"])

    def quadrature(self) -> FrequencyQuadrature:
        return FrequencyQuadrature(self._get(2, np.float64).reshape(-1, 2),
                                   self._get(3, np.float64).view(np.complex128),
                                   self._get(7, np.int32))

    def close_matrix(self) -> SparsePairMatrix:
        return SparsePairMatrix(self._get(4, np.uint64), self._get(5, np.uint32),
                                self._get(6, np.float64).view(np.complex128))

    def kernel(self) -> KernelSpec:
        i = self.info()
        return KernelSpec("helmholtz" if i["kind"] == 1 else "laplace", i["k"])

    def eps(self) -> float:
        return self.info()["eps"]

    def delta_min(self) -> float:
        return self.info()["delta_min"]

    def delta_max(self) -> float:
        return self.info()["delta_max"]

    def annulus_a(self) -> float:
        return self.info()["a"]

    def bytes(self) -> int:
        return int(self.info()["bytes"])

    # -- the hot path
    def apply(self, f) -> np.ndarray:
        """q = A f (conv_operator.cpp:301-309). f: (n_src,) or (nrhs, n_src)."""
        return self._host_apply(f, adjoint=False)

    def apply_adjoint(self, u) -> np.ndarray:
        """q = A^H u (conv_operator.cpp:311-324)."""
        return self._host_apply(u, adjoint=True)

    def _host_apply(self, x, adjoint: bool) -> np.ndarray:
        info = self.info()
        n_in, n_out = (info["n_tgt"], info["n_src"]) if adjoint else (info["n_src"], info["n_tgt"])
        x = _cx(x)
        batched = x.ndim == 2
        xb = x.reshape(-1, x.shape[-1]) if x.ndim else x
        if xb.shape[-1] != n_in:
            raise ValueError(("apply_adjoint" if adjoint else "apply") + ": input size mismatch")
        nrhs = xb.shape[0]
        out = np.empty((nrhs, n_out), np.complex128)
        fn = lib.sbd_op_apply_adjoint if adjoint else lib.sbd_op_apply
        check(fn(self._h, xb.view(np.float64).ctypes.data_as(_dp),
                 out.view(np.float64).ctypes.data_as(_dp), nrhs))
        return out if batched else out[0]

    def apply_device(self, f_ptr: int, q_ptr: int, nrhs: int = 1, stream: int = 0,
                     f_is_real=None) -> None:
        """Device-buffer apply (interleaved complex128, nrhs x n). Enqueued on
        `stream` (a cudaStream_t as int; 0 = the legacy default stream); never
        synchronises. f_is_real: None (unknown, decided on the device), a bool
        for every column, or a list of nrhs bools (sbd_op_apply_device_ex)."""
        if f_is_real is None:
            check(lib.sbd_op_apply_device(self._h, ctypes.c_void_p(f_ptr), ctypes.c_void_p(q_ptr),
                                          int(nrhs), ctypes.c_void_p(stream or None)))
            return
        flags = [f_is_real] * nrhs if isinstance(f_is_real, (bool, int)) else list(f_is_real)
        arr = (ctypes.c_int * nrhs)(*[1 if x else 0 for x in flags])
        check(lib.sbd_op_apply_device_ex(self._h, ctypes.c_void_p(f_ptr), ctypes.c_void_p(q_ptr),
                                         int(nrhs), ctypes.c_void_p(stream or None), arr))

    def apply_host(self, f_ptr: int, q_ptr: int, nrhs: int = 1) -> None:
        """sbd_op_apply on raw host pointers (e.g. pinned torch buffers)."""
        check(lib.sbd_op_apply(self._h, ctypes.cast(f_ptr, _dp), ctypes.cast(q_ptr, _dp),
                               int(nrhs)))

    def apply_async(self, f_ptr: int, q_ptr: int, nrhs: int = 1) -> int:
        """sbd_op_apply_async on raw host pointers; returns the ticket for wait()."""
        t = ctypes.c_uint64()
        check(lib.sbd_op_apply_async(self._h, ctypes.cast(f_ptr, _dp), ctypes.cast(q_ptr, _dp), int(nrhs),
                                     ctypes.byref(t)))
        return t.value

    def wait(self, ticket: int) -> None:
        check(lib.sbd_op_wait(self._h, int(ticket)))

    def apply_adjoint_device(self, u_ptr: int, q_ptr: int, nrhs: int = 1, stream: int = 0) -> None:
        check(lib.sbd_op_apply_adjoint_device(self._h, ctypes.c_void_p(u_ptr),
                                              ctypes.c_void_p(q_ptr), int(nrhs),
                                              ctypes.c_void_p(stream or None)))

    def set_profiling(self, on: bool) -> None:
        check(lib.sbd_op_set_profiling(self._h, 1 if on else 0))

    def stage_times(self, reset: bool = True) -> list:
        """(stage, ms) for every profiled stage launch since the last reset."""
        cap = 4096
        ms = (ctypes.c_double * cap)()
        names = (ctypes.c_char_p * cap)()
        n = lib.sbd_op_stage_times(self._h, ms, names, cap)
        out = [(names[i].decode(), ms[i]) for i in range(min(n, cap))]
        if reset:
            check(lib.sbd_op_stage_times_reset(self._h))
        return out


# --------------------------------------------------------------- NUFFT
@dataclasses.dataclass
class NufftOptions:
    """nufft.hpp:18-24."""
    tol: float = 1e-9
    mode: str = "auto"  # auto | direct | fast
    direct_threshold: int = 1 << 20
    max_grid_bytes: int = 4 << 30
    device: int = 0


PLUS, MINUS = +1, -1


class NufftPlan:
    """nufft.hpp:30-56: type-III plan, apply / apply_transpose on the GPU."""

    def __init__(self, points, freqs, sign: int, options: Optional[NufftOptions] = None):
        o = options or NufftOptions()
        p, f = _xy(points), _xy(freqs)
        self.np, self.nf = len(p), len(f)
        mode = {"auto": 0, "direct": 1, "fast": 2}[o.mode]
        h = ctypes.c_void_p()
        check(lib.sbd_nufft_create(_ptr(p), len(p), _ptr(f), len(f), int(sign), float(o.tol),
                                   mode, int(o.direct_threshold), int(o.max_grid_bytes),
                                   int(o.device), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            lib.sbd_nufft_destroy(self._h)
            self._h = None

    def _meta(self):
        fast, w, n1, n2 = (ctypes.c_int() for _ in range(4))
        check(lib.sbd_nufft_info(self._h, ctypes.byref(fast), ctypes.byref(w), ctypes.byref(n1),
                                 ctypes.byref(n2)))
        return fast.value, w.value, n1.value, n2.value

    def fast_path(self) -> bool:
        return bool(self._meta()[0])

    def kernel_width(self) -> int:
        return self._meta()[1]

    def grid_cells(self) -> int:
        fast, _, n1, n2 = self._meta()
        return n1 * n2 if fast else 0

    def apply(self, coeffs) -> np.ndarray:
        c = _cx(coeffs)
        if c.shape != (self.np,):
            raise ValueError("nufft apply: coefficient count mismatch")
        out = np.empty(self.nf, np.complex128)
        check(lib.sbd_nufft_apply(self._h, c.view(np.float64).ctypes.data_as(_dp),
                                  out.view(np.float64).ctypes.data_as(_dp)))
        return out

    def apply_transpose(self, values) -> np.ndarray:
        v = _cx(values)
        if v.shape != (self.nf,):
            raise ValueError("nufft apply_transpose: value count mismatch")
        out = np.empty(self.np, np.complex128)
        check(lib.sbd_nufft_apply_transpose(self._h, v.view(np.float64).ctypes.data_as(_dp),
                                            out.view(np.float64).ctypes.data_as(_dp)))
        return out


def ndft_direct(points, freqs, coeffs, sign: int, device: int = 0) -> np.ndarray:
    """nufft.cpp:76-93 on the GPU."""
    p, f, c = _xy(points), _xy(freqs), _cx(coeffs)
    if len(c) != len(p):
        raise ValueError("ndft_direct: points/coeffs size mismatch")
    out = np.empty(len(f), np.complex128)
    check(lib.sbd_ndft_direct(_ptr(p), len(p), _ptr(f), len(f),
                              c.view(np.float64).ctypes.data_as(_dp), int(sign), int(device),
                              out.view(np.float64).ctypes.data_as(_dp)))
    return out
