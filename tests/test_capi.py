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
