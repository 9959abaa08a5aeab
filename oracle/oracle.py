"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (ctypes bindings to the checkers).

Two CPU checkers live under oracle/:

* ``RefLib`` binds ``oracle/_ref/libsbdref.so``: the UNMODIFIED reference
  library (/root/reference/proj/src) compiled against the test-only shims in
  oracle/shim/ by oracle/Makefile, plus oracle/ref_driver.cpp. This is the
  reference itself; it pins everything else.
* ``Oracle`` binds ``oracle/liboracle.so``: the plain-C restatement of the
  apply path (oracle/sbd_oracle.c), which needs nothing from /root/reference and
  is pinned against ``RefLib`` and the golden fixtures in tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsbdref.so")
ORACLE_SO = os.path.join(HERE, "liboracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_u64 = ctypes.c_uint64


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def as_xy(points) -> np.ndarray:
    """(n, 2) float64 C-contiguous."""
    a = np.ascontiguousarray(points, dtype=np.float64)
    return a.reshape(-1, 2)


def as_cplx(v) -> np.ndarray:
    """complex128 C-contiguous (interleaved re, im in memory)."""
    return np.ascontiguousarray(v, dtype=np.complex128).reshape(-1)


class Oracle:
    """Plain-C restatement (oracle/sbd_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle liboracle.so`")
        L = ctypes.CDLL(path)
        L.orc_last_error.restype = ctypes.c_char_p
        L.orc_bessel_i0.restype = ctypes.c_double
        L.orc_bessel_i0.argtypes = [ctypes.c_double]
        L.orc_kb_window.restype = ctypes.c_double
        L.orc_kb_window.argtypes = [ctypes.c_double, ctypes.c_double]
        L.orc_kb_window_hat.restype = ctypes.c_double
        L.orc_kb_window_hat.argtypes = [ctypes.c_double, ctypes.c_double]
        L.orc_plan_create.restype = ctypes.c_void_p
        L.orc_plan_create.argtypes = [_dp, _u64, _dp, _u64, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_int, _u64, _u64]
        L.orc_plan_free.argtypes = [ctypes.c_void_p]
        L.orc_plan_apply.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc_plan_apply_transpose.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc_plan_geometry.argtypes = [ctypes.c_void_p, _dp]
        L.orc_ndft_direct.argtypes = [_dp, _u64, _dp, _u64, _dp, ctypes.c_int, _dp]
        L.orc_op_open.restype = ctypes.c_void_p
        L.orc_op_open.argtypes = [ctypes.c_char_p, _u64]
        L.orc_op_free.argtypes = [ctypes.c_void_p]
        L.orc_op_info.argtypes = [ctypes.c_void_p, _dp]
        L.orc_op_apply.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc_op_apply_adjoint.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc_op_stage.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc_op_weights.argtypes = [ctypes.c_void_p, _dp]
        self.L = L

    def err(self):
        return self.L.orc_last_error().decode()

    def ndft_direct(self, points, freqs, coeffs, sign):
        p, f, c = as_xy(points), as_xy(freqs), as_cplx(coeffs)
        out = np.zeros(len(f), np.complex128)
        self.L.orc_ndft_direct(_p(p), len(p), _p(f), len(f), _p(c.view(np.float64)), int(sign),
                               _p(out.view(np.float64)))
        return out

    def plan(self, points, freqs, sign, tol, mode=0, direct_threshold=1 << 20,
             max_grid_bytes=4 << 30):
        return OraclePlan(self, points, freqs, sign, tol, mode, direct_threshold, max_grid_bytes)

    def op(self, path, max_grid_bytes=0):
        return OracleOp(self, path, max_grid_bytes)


class OraclePlan:
    def __init__(self, o, points, freqs, sign, tol, mode, direct_threshold, max_grid_bytes):
        self.o = o
        p, f = as_xy(points), as_xy(freqs)
        self.np, self.nf = len(p), len(f)
        self.h = o.L.orc_plan_create(_p(p), len(p), _p(f), len(f), int(sign), float(tol),
                                     int(mode), int(direct_threshold), int(max_grid_bytes))
        if not self.h:
            raise RuntimeError(o.err())

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_plan_free(self.h)
            self.h = None

    def geometry(self):
        g = np.zeros(12)
        self.o.L.orc_plan_geometry(self.h, _p(g))
        keys = ["fast", "w", "beta", "n1", "n2", "cx", "cy", "fcx", "fcy", "gx", "gy", "cells"]
        return dict(zip(keys, g.tolist()))

    def apply(self, coeffs):
        c = as_cplx(coeffs)
        assert len(c) == self.np
        out = np.zeros(self.nf, np.complex128)
        self.o.L.orc_plan_apply(self.h, _p(c.view(np.float64)), _p(out.view(np.float64)))
        return out

    def apply_transpose(self, values):
        v = as_cplx(values)
        assert len(v) == self.nf
        out = np.zeros(self.np, np.complex128)
        self.o.L.orc_plan_apply_transpose(self.h, _p(v.view(np.float64)), _p(out.view(np.float64)))
        return out


class OracleOp:
    def __init__(self, o, path, max_grid_bytes=0):
        self.o = o
        self.h = o.L.orc_op_open(path.encode(), int(max_grid_bytes))
        if not self.h:
            raise RuntimeError(o.err())
        info = np.zeros(10)
        o.L.orc_op_info(self.h, _p(info))
        self.n_src, self.n_tgt, self.n_xi, self.nnz = (int(x) for x in info[:4])
        self.single = bool(info[4])

    def __del__(self):
        if getattr(self, "h", None):
            self.o.L.orc_op_free(self.h)
            self.h = None

    def apply(self, f):
        f = as_cplx(f)
        assert len(f) == self.n_src
        q = np.zeros(self.n_tgt, np.complex128)
        if self.o.L.orc_op_apply(self.h, _p(f.view(np.float64)), _p(q.view(np.float64))):
            raise RuntimeError(self.o.err())
        return q

    def apply_adjoint(self, u):
        u = as_cplx(u)
        assert len(u) == self.n_tgt
        q = np.zeros(self.n_src, np.complex128)
        if self.o.L.orc_op_apply_adjoint(self.h, _p(u.view(np.float64)), _p(q.view(np.float64))):
            raise RuntimeError(self.o.err())
        return q

    def weights(self):
        w = np.zeros(self.n_xi, np.complex128)
        self.o.L.orc_op_weights(self.h, _p(w.view(np.float64)))
        return w

    def stage(self, stage, x, out=None):
        x = as_cplx(x)
        n_out = {1: self.n_xi, 2: self.n_tgt, 3: self.n_tgt}[stage]
        out = np.zeros(n_out, np.complex128) if out is None else as_cplx(out).copy()
        if self.o.L.orc_op_stage(self.h, stage, _p(x.view(np.float64)), _p(out.view(np.float64))):
            raise RuntimeError(self.o.err())
        return out


class RefLib:
    """The unmodified reference, compiled into oracle/_ref/libsbdref.so."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` (needs /root/reference)")
        L = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_assemble_save.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _u64, _dp, _u64,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, _u64, ctypes.c_char_p, _dp]
        L.ref_op_load.restype = ctypes.c_void_p
        L.ref_op_load.argtypes = [ctypes.c_char_p]
        L.ref_op_free.argtypes = [ctypes.c_void_p]
        L.ref_op_apply.argtypes = [ctypes.c_void_p, _dp, _u64, _dp]
        L.ref_op_apply_adjoint.argtypes = [ctypes.c_void_p, _dp, _u64, _dp]
        L.ref_raw_open.restype = ctypes.c_void_p
        L.ref_raw_open.argtypes = [ctypes.c_char_p, _u64]
        L.ref_raw_free.argtypes = [ctypes.c_void_p]
        L.ref_raw_stage.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _u64, _dp]
        L.ref_nufft.argtypes = [_dp, _u64, _dp, _u64, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                _u64, ctypes.c_int, _dp, _dp, ctypes.POINTER(ctypes.c_int)]
        L.ref_bessel.restype = ctypes.c_double
        L.ref_bessel.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double]
        L.ref_cloud_diameter.restype = ctypes.c_double
        L.ref_cloud_diameter.argtypes = [_dp, _u64]
        L.ref_choose_parameters.argtypes = [_u64, ctypes.c_double, ctypes.c_double, _dp,
                                            ctypes.POINTER(ctypes.c_int)]
        self.L = L

    def err(self):
        return self.L.ref_last_error().decode()

    def assemble_save(self, path, src, tgt=None, kind=0, k=0.0, eps=1e-6, alpha=0.0,
                      a_override=0.0, small_k_factor=0.5, max_grid_bytes=0):
        s = as_xy(src)
        t = None if tgt is None else as_xy(tgt)
        info = np.zeros(8)
        rc = self.L.ref_assemble_save(int(kind), float(k), _p(s), len(s), _p(t),
                                      0 if t is None else len(t), float(eps), float(alpha),
                                      float(a_override), float(small_k_factor),
                                      int(max_grid_bytes), path.encode(), _p(info))
        if rc:
            raise {1: ValueError, 2: ValueError}.get(rc, RuntimeError)(self.err())
        keys = ["a", "dmin", "dmax", "P", "n_xi", "nnz", "bytes", "sbd_error"]
        return dict(zip(keys, info.tolist()))

    def load(self, path):
        return RefOp(self, path)

    def raw(self, path, max_grid_bytes=0):
        return RefRaw(self, path, max_grid_bytes)

    def nufft(self, points, freqs, coeffs, sign, tol, mode=0, transpose=False,
              max_grid_bytes=0):
        p, f = as_xy(points), as_xy(freqs)
        c = as_cplx(coeffs)
        out = np.zeros(len(p) if transpose else len(f), np.complex128)
        meta = (ctypes.c_int * 2)()
        rc = self.L.ref_nufft(_p(p), len(p), _p(f), len(f), int(sign), float(tol), int(mode),
                              int(max_grid_bytes), int(transpose), _p(c.view(np.float64)),
                              _p(out.view(np.float64)), meta)
        if rc:
            raise RuntimeError(self.err())
        return out, {"fast": meta[0], "w": meta[1]}

    def bessel(self, which, x, n=0):
        idx = {"j0": 0, "j1": 1, "jn": 2, "y0": 3, "y1": 4, "i0": 5}[which]
        return self.L.ref_bessel(idx, int(n), float(x))

    def diameter(self, points):
        p = as_xy(points)
        return self.L.ref_cloud_diameter(_p(p), len(p))

    def choose_parameters(self, n, eps, alpha):
        a = ctypes.c_double()
        ph = ctypes.c_int()
        if self.L.ref_choose_parameters(int(n), float(eps), float(alpha), ctypes.byref(a),
                                        ctypes.byref(ph)):
            raise ValueError(self.err())
        return a.value, ph.value


class RefOp:
    def __init__(self, lib, path):
        self.lib = lib
        self.h = lib.L.ref_op_load(path.encode())
        if not self.h:
            raise RuntimeError(lib.err())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_op_free(self.h)
            self.h = None

    def apply(self, f, n_out=None):
        f = as_cplx(f)
        q = np.zeros(n_out or len(f), np.complex128)
        if self.lib.L.ref_op_apply(self.h, _p(f.view(np.float64)), len(f), _p(q.view(np.float64))):
            raise ValueError(self.lib.err())
        return q

    def apply_adjoint(self, u, n_out):
        u = as_cplx(u)
        q = np.zeros(n_out, np.complex128)
        if self.lib.L.ref_op_apply_adjoint(self.h, _p(u.view(np.float64)), len(u),
                                           _p(q.view(np.float64))):
            raise ValueError(self.lib.err())
        return q


class RefRaw:
    """The reference's own NufftPlan / SparsePairMatrix driven stage by stage."""

    def __init__(self, lib, path, max_grid_bytes=0):
        self.lib = lib
        self.h = lib.L.ref_raw_open(path.encode(), int(max_grid_bytes))
        if not self.h:
            raise RuntimeError(lib.err())

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.L.ref_raw_free(self.h)
            self.h = None

    def stage(self, stage, x, n_out, out=None):
        x = as_cplx(x)
        out = np.zeros(n_out, np.complex128) if out is None else as_cplx(out).copy()
        if self.lib.L.ref_raw_stage(self.h, int(stage), _p(x.view(np.float64)), len(x),
                                    _p(out.view(np.float64))):
            raise RuntimeError(self.lib.err())
        return out

    def apply(self, f, n_out):
        return self.stage(0, f, n_out)
