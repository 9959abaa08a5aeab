"""CPU: the C-ABI library loads, exports every symbol include/sbd_b200.h
declares, and its host-only entry points behave like the reference (no compute
calls: there is no GPU here)."""
import ctypes
import os
import re

import numpy as np
import pytest

from tests.conftest import GOLDEN, ROOT

import paper_1711_07877_b200 as sbd
from paper_1711_07877_b200 import _capi


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "sbd_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(sbd_[a-z0-9_]+)\s*\(", txt)))


def test_library_loads_and_exports_header_symbols():
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_capi.EXPORTED) == syms


def test_version_string():
    assert b"sm_100a" in _capi.lib.sbd_version()


def test_choose_parameters_formula_and_guards():
    # test_operator.cpp:14-33
    a, ph = sbd.choose_parameters(1_000_000, 1e-6, 0.0)
    assert abs(a - abs(np.log(1e-6)) ** (2 / 3) / 1e6 ** (2 / 3)) < 1e-18
    assert ph > 0
    prev = 1.0
    for n in (100, 1000, 10000, 100000):
        a, _ = sbd.choose_parameters(n, 1e-6, 0.0)
        assert a < prev
        prev = a
    assert sbd.choose_parameters(10000, 1e-6, 1 / 6)[0] > sbd.choose_parameters(10000, 1e-6, 0)[0]
    assert sbd.choose_parameters(20, 1e-3, 0.0)[0] <= 0.5
    with pytest.raises(sbd.DomainError):
        sbd.choose_parameters(5, 1e-3, 0.0)
    with pytest.raises(sbd.DomainError):
        sbd.choose_parameters(100, 1e-3, 0.4)


def test_choose_parameters_matches_reference(reflib):
    for n, eps, al in [(10**4, 1e-6, 0.0), (10**6, 1e-6, 0.0), (12345, 1e-3, 1 / 6)]:
        assert sbd.choose_parameters(n, eps, al) == reflib.choose_parameters(n, eps, al)


def test_load_errors_before_any_device_work(tmp_path):
    with pytest.raises(sbd.SbdError, match="cannot open"):
        sbd.CompressedOperator.load(str(tmp_path / "missing.sbdop"))
    bad = tmp_path / "bad.sbdop"
    bad.write_bytes(b"NOTSBDOP" + b"\0" * 64)
    with pytest.raises(sbd.SbdError, match="bad magic"):
        sbd.CompressedOperator.load(str(bad))
    trunc = tmp_path / "trunc.sbdop"
    trunc.write_bytes(open(os.path.join(GOLDEN, "lap_disk_n1000.sbdop"), "rb").read()[:5000])
    with pytest.raises(sbd.SbdError, match="truncated"):
        sbd.CompressedOperator.load(str(trunc))


def _sbdop_offsets(buf):
    """Byte offsets of the arrays of an SBDOPv1 file (conv_operator.cpp:357-397)."""
    import struct
    off = 8 + 4 + 8
    single = buf[off]
    off += 1 + 6 * 8
    out = {}

    def vec(name, esz):
        nonlocal off
        n = struct.unpack_from("<Q", buf, off)[0]
        out[name] = (off + 8, n)
        off += 8 + n * esz

    vec("src", 16)
    off += 8
    if not single:
        vec("tgt", 16)
        off += 8
    vec("freqs", 16)
    vec("weights", 16)
    vec("ring_offsets", 4)
    off += 8
    vec("row_offsets", 8)
    vec("cols", 4)
    vec("values", 16)
    return out


@pytest.mark.parametrize("field,value,what", [("cols", 10**6, "column index"),
                                              ("row_offsets", 2**40, "row offsets"),
                                              ("ring_offsets", 10**9, "ring offsets")])
def test_load_rejects_inconsistent_csr_and_rings(tmp_path, field, value, what):
    # a foreign or corrupt file must fail at load time, before any
    # array reaches the device (an out-of-range column would otherwise read
    # out of bounds in the SpMV kernels)
    import struct
    buf = bytearray(open(os.path.join(GOLDEN, "lap_disk_n1000.sbdop"), "rb").read())
    start, n = _sbdop_offsets(buf)[field]
    k = n // 2
    fmt = {"cols": "<I", "row_offsets": "<Q", "ring_offsets": "<i"}[field]
    struct.pack_into(fmt, buf, start + k * struct.calcsize(fmt), value)
    bad = tmp_path / "bad.sbdop"
    bad.write_bytes(bytes(buf))
    with pytest.raises(sbd.SbdError, match=what):
        sbd.CompressedOperator.load(str(bad))


def test_op_options_are_checked():
    # sbd_op_options replaces the r1 environment switches; bad values are
    # rejected before any file is read
    oc = sbd.OpOptions()._c()
    oc.spread_kernel = 7
    h = ctypes.c_void_p()
    rc = _capi.lib.sbd_op_load_ex(os.path.join(GOLDEN, "lap_disk_n1000.sbdop").encode(), 0, 0,
                                  ctypes.byref(oc), ctypes.byref(h))
    assert rc == 1 and b"options" in _capi.lib.sbd_last_error()
    d = _capi.OpOptionsC()
    _capi.lib.sbd_op_options_default(ctypes.byref(d))
    assert (d.real_input_split, d.hermitian_fft, d.radix_first_pass, d.fused) == (1, 1, -1, 1)


def test_no_environment_switches_in_the_library():
    # no process-wide getenv knobs inside the drop-in library
    import glob
    for path in glob.glob(os.path.join(ROOT, "paper_1711_07877_b200", "csrc", "*")):
        assert "getenv" not in open(path).read(), path


@pytest.mark.parametrize("w", list(range(4, 18)))
def test_window_polynomial_accuracy(w):
    # The device KB window (degree-15 per-tap polynomials) must match
    # I0(beta sqrt(1-z^2)) to ~1e-16 of its peak for every width the
    # reference can select (nufft.cpp:47-52, beta = 2.3562 w, :129).
    err = _capi.lib.sbd_window_fit_error(w, 2.3562 * w)
    assert 0 <= err <= 2e-15, err


def test_host_bessel_vs_reference(reflib):
    # The offline assembly's J0/J1/Y0/Y1 against the reference's (bessel.cpp),
    # across the series / float128 / Hankel seams.
    xs = np.concatenate([np.linspace(1e-3, 30, 997), np.geomspace(30, 2e4, 300)])
    for which, name in enumerate(["j0", "j1", "y0", "y1"]):
        got = np.array([_capi.lib.sbd_bessel(which, x) for x in xs])
        want = np.array([reflib.bessel(name, x) for x in xs])
        scale = np.maximum(np.abs(want), 1.0 / np.sqrt(xs))  # absolute near zeros
        assert np.max(np.abs(got - want) / scale) <= 5e-14, name


def test_host_bessel_golden_mpmath():
    # 50-digit values (mpmath) at a few arguments, independent of the reference.
    import mpmath as mp
    mp.mp.dps = 30
    for x in (0.1, 2.5, 11.9, 12.1, 15.9, 16.1, 100.0, 1234.5):
        for which, f in enumerate([lambda t: mp.besselj(0, t), lambda t: mp.besselj(1, t),
                                   lambda t: mp.bessely(0, t), lambda t: mp.bessely(1, t)]):
            want = float(f(x))
            got = _capi.lib.sbd_bessel(which, x)
            assert abs(got - want) <= 2e-15 * max(abs(want), 1.0 / np.sqrt(x)), (which, x)
