"""ctypes binding of include/sbd_b200.h (the C ABI of libsbd_b200.so).

Importing this module loads the in-tree native library and fails loudly if it
is missing: there is no CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsbd_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python paper_1711_07877_b200/build.py` "
        "(the SBD apply path has no CPU fallback)")

lib = ctypes.CDLL(LIB_PATH)

_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_int = ctypes.c_int


class OpOptionsC(ctypes.Structure):
    _fields_ = [("real_input_split", _int), ("hermitian_fft", _int), ("radix_first_pass", _int),
                ("spread_kernel", _int), ("interp_kernel", _int), ("fused", _int), ("verbose", _int),
                ("procedural_rings", _int)]


class AssembleOptionsC(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double), ("alpha", ctypes.c_double),
                ("a_override", ctypes.c_double), ("small_k_factor", ctypes.c_double),
                ("nufft_direct_threshold", _u64), ("max_grid_bytes", _u64), ("device", _int),
                ("pipeline", OpOptionsC)]


class OpInfoC(ctypes.Structure):
    _fields_ = [("n_src", _u64), ("n_tgt", _u64), ("n_xi", _u64), ("nnz", _u64),
                ("single_cloud", _int), ("kind", _int),
                ("k", ctypes.c_double), ("eps", ctypes.c_double), ("alpha", ctypes.c_double),
                ("a", ctypes.c_double), ("delta_min", ctypes.c_double),
                ("delta_max", ctypes.c_double), ("nufft_tol", ctypes.c_double),
                ("P", _int), ("w", _int), ("beta", ctypes.c_double),
                ("n1_in", _int), ("n2_in", _int), ("n1_out", _int), ("n2_out", _int),
                ("fast_in", _int), ("fast_out", _int),
                ("bytes", _u64), ("device_bytes", _u64), ("procedural_rings", _int)]


def _sig(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("sbd_last_error", ctypes.c_char_p)
_sig("sbd_version", ctypes.c_char_p)
_sig("sbd_kernel_launch_count", _u64)
_sig("sbd_assemble_options_default", None, ctypes.POINTER(AssembleOptionsC))
_sig("sbd_op_options_default", None, ctypes.POINTER(OpOptionsC))
_sig("sbd_op_assemble", _int, _int, ctypes.c_double, _dp, _u64, _dp, _u64,
     ctypes.POINTER(AssembleOptionsC), ctypes.POINTER(_vp))
_sig("sbd_op_load", _int, ctypes.c_char_p, _int, _u64, ctypes.POINTER(_vp))
_sig("sbd_op_load_ex", _int, ctypes.c_char_p, _int, _u64, ctypes.POINTER(OpOptionsC), ctypes.POINTER(_vp))
_sig("sbd_op_save", _int, _vp, ctypes.c_char_p)
_sig("sbd_op_destroy", _int, _vp)
_sig("sbd_op_info", _int, _vp, ctypes.POINTER(OpInfoC))
_sig("sbd_op_get", _int, _vp, _int, _vp, ctypes.POINTER(_u64))
_sig("sbd_op_apply", _int, _vp, _dp, _dp, _int)
_sig("sbd_op_apply_adjoint", _int, _vp, _dp, _dp, _int)
_sig("sbd_op_apply_async", _int, _vp, _dp, _dp, _int, ctypes.POINTER(_u64))
_sig("sbd_op_wait", _int, _vp, _u64)
_sig("sbd_op_apply_device", _int, _vp, _vp, _vp, _int, _vp)
_sig("sbd_op_apply_device_ex", _int, _vp, _vp, _vp, _int, _vp, ctypes.POINTER(_int))
_sig("sbd_op_apply_adjoint_device", _int, _vp, _vp, _vp, _int, _vp)
_sig("sbd_op_set_profiling", _int, _vp, _int)
_sig("sbd_op_shard_bounds", _int, _vp, _int, _int, ctypes.POINTER(_u64))
_sig("sbd_op_forward_spectrum", _int, _vp, _vp, _u64, _u64, _vp, _vp)
_sig("sbd_op_backward_targets", _int, _vp, _vp, _vp, _u64, _u64, _vp, _vp)
_sig("sbd_op_spectrum_length", _int, _vp, _vp, _vp, ctypes.POINTER(_u64))
_sig("sbd_op_stage_times", _int, _vp, _dp, ctypes.POINTER(ctypes.c_char_p), _int)
_sig("sbd_slab_create", _int, _vp, _int, _int, ctypes.POINTER(_vp))
_sig("sbd_slab_destroy", _int, _vp)
_sig("sbd_slab_counts", _int, _vp, _int, ctypes.POINTER(_u64), ctypes.POINTER(_u64))
_sig("sbd_slab_stage", _int, _vp, _int, _vp, _vp, _vp, _vp)
_sig("sbd_op_stage_times_reset", _int, _vp)
_sig("sbd_cloud_diameter", ctypes.c_double, _dp, _u64)
_sig("sbd_nufft_create", _int, _dp, _u64, _dp, _u64, _int, ctypes.c_double, _int, _u64, _u64,
     _int, ctypes.POINTER(_vp))
_sig("sbd_nufft_apply", _int, _vp, _dp, _dp)
_sig("sbd_nufft_apply_transpose", _int, _vp, _dp, _dp)
_sig("sbd_nufft_info", _int, _vp, ctypes.POINTER(_int), ctypes.POINTER(_int),
     ctypes.POINTER(_int), ctypes.POINTER(_int))
_sig("sbd_nufft_destroy", _int, _vp)
_sig("sbd_ndft_direct", _int, _dp, _u64, _dp, _u64, _dp, _int, _int, _dp)
_sig("sbd_window_fit_error", ctypes.c_double, _int, ctypes.c_double)
_sig("sbd_bessel", ctypes.c_double, _int, ctypes.c_double)
_sig("sbd_choose_parameters", _int, _u64, ctypes.c_double, ctypes.c_double, _dp,
     ctypes.POINTER(_int))

# The symbols include/sbd_b200.h declares (checked by tests/test_capi_symbols.py).
EXPORTED = [
    "sbd_last_error", "sbd_version", "sbd_assemble_options_default", "sbd_op_options_default",
    "sbd_op_assemble", "sbd_op_load", "sbd_op_load_ex", "sbd_op_save", "sbd_op_destroy", "sbd_op_info", "sbd_op_get",
    "sbd_op_apply", "sbd_op_apply_adjoint", "sbd_op_apply_async", "sbd_op_wait",
    "sbd_op_apply_device", "sbd_op_apply_device_ex",
    "sbd_op_apply_adjoint_device", "sbd_op_set_profiling", "sbd_op_stage_times",
    "sbd_op_stage_times_reset", "sbd_cloud_diameter",
    "sbd_nufft_create", "sbd_nufft_apply", "sbd_nufft_apply_transpose", "sbd_nufft_info",
    "sbd_nufft_destroy", "sbd_ndft_direct", "sbd_choose_parameters", "sbd_kernel_launch_count",
    "sbd_window_fit_error", "sbd_bessel", "sbd_op_shard_bounds", "sbd_op_forward_spectrum",
    "sbd_op_backward_targets", "sbd_op_spectrum_length",
    "sbd_slab_create", "sbd_slab_destroy", "sbd_slab_counts", "sbd_slab_stage",
]


class SbdError(RuntimeError):
    """Base class for errors raised by the native layer."""


class DomainError(ValueError):
    """std::domain_error analogue (conv_operator.cpp:122-127, 265)."""


class CudaError(SbdError):
    """CUDA / cuFFT failure (no reference analogue)."""


class SbdConvergenceError(SbdError):
    """SbdConvergenceError analogue (sbd.hpp:31-38)."""


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = lib.sbd_last_error().decode(errors="replace")
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise DomainError(msg)
    if rc == 4:
        raise CudaError(msg)
    if rc == 5:
        raise SbdConvergenceError(msg)
    raise SbdError(msg)


def launch_count() -> int:
    return int(lib.sbd_kernel_launch_count())
