"""CPU: pin the plain-C restatement (oracle/sbd_oracle.c) against the golden
fixtures generated from the unmodified reference, and -- where the compiled
reference (oracle/_ref) is present -- against the reference itself."""
import numpy as np
import pytest

from tests.conftest import GOLDEN, golden, golden_cases, rel_l2

CASES = [c["name"] for c in golden_cases()]


def test_bessel_i0_kat(oracle):
    kat = np.load(f"{GOLDEN}/nufft_kat.npz")
    got = np.array([oracle.L.orc_bessel_i0(float(x)) for x in kat["i0_x"]])
    assert np.array_equal(got, kat["i0"])  # same series, same order: bit-exact


@pytest.mark.parametrize("tol", [1e-4, 1e-8, 1e-12])
@pytest.mark.parametrize("sign", [-1, 1])
def test_nufft_kat(oracle, tol, sign):
    kat = np.load(f"{GOLDEN}/nufft_kat.npz")
    key = f"tol{tol:.0e}_s{'p' if sign > 0 else 'm'}"
    plan = oracle.plan(kat["pts"], kat["frq"], sign, tol, mode=2)
    a = plan.apply(kat["c"])
    t = plan.apply_transpose(kat["v"])
    # restatement of the reference arithmetic: agreement to a few ulps
    assert np.max(np.abs(a - kat["apply_" + key])) <= 1e-13 * np.abs(kat["c"]).sum()
    assert np.max(np.abs(t - kat["transpose_" + key])) <= 1e-13 * np.abs(kat["v"]).sum()
    # and the reference's own accuracy contract vs the exact sum (test_nufft.cpp:63-92)
    d = oracle.ndft_direct(kat["pts"], kat["frq"], kat["c"], sign)
    assert np.max(np.abs(a - d)) <= tol * np.abs(kat["c"]).sum()


def test_ndft_direct_kat(oracle):
    kat = np.load(f"{GOLDEN}/nufft_kat.npz")
    d = oracle.ndft_direct(kat["pts"], kat["frq"], kat["c"], +1)
    assert np.max(np.abs(d - kat["direct_p"])) <= 1e-13 * np.abs(kat["c"]).sum()


def test_ndft_direct_sign_convention(oracle):
    # test_nufft.cpp:38-45: e^{+i z.xi} for Plus, e^{-i z.xi} for Minus
    z, xi = np.array([[0.3, -1.1]]), np.array([[2.0, 5.0]])
    ph = 0.3 * 2.0 - 1.1 * 5.0
    assert abs(oracle.ndft_direct(z, xi, [1.0], +1)[0] - np.exp(1j * ph)) < 1e-15
    assert abs(oracle.ndft_direct(z, xi, [1.0], -1)[0] - np.exp(-1j * ph)) < 1e-15


@pytest.mark.parametrize("name", CASES)
def test_operator_golden(oracle, name):
    path, g = golden(name)
    op = oracle.op(path)
    assert rel_l2(op.apply(g["f"]), g["q"]) <= 1e-13
    assert rel_l2(op.apply_adjoint(g["u"]), g["qa"]) <= 1e-13
    assert rel_l2(op.stage(1, g["f"]), g["spectrum"]) <= 1e-13


@pytest.mark.parametrize("name", CASES[:3])
def test_operator_vs_reference_random(oracle, reflib, name):
    path, g = golden(name)
    rng = np.random.default_rng(99)
    f = rng.standard_normal(len(g["f"])) + 1j * rng.standard_normal(len(g["f"]))
    want = reflib.load(path).apply(f, len(g["q"]))
    got = oracle.op(path).apply(f)
    assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))


def test_plan_geometry_matches_reference_widths(oracle, reflib):
    rng = np.random.default_rng(3)
    pts = rng.uniform(-1, 1, (64, 2))
    frq = rng.uniform(-60, 60, (75, 2))
    for tol in (1e-3, 1e-6, 1e-9, 1e-14):
        _, meta = reflib.nufft(pts, frq, np.ones(64), +1, tol, mode=2)
        geo = oracle.plan(pts, frq, +1, tol, mode=2).geometry()
        assert meta["w"] == geo["w"]


def test_grid_guard(oracle):
    # test_nufft.cpp:193-203: the grid-memory guard refuses oversized grids
    rng = np.random.default_rng(43)
    pts, frq = rng.uniform(-.5, .5, (64, 2)), rng.uniform(-2500, 2500, (64, 2))
    with pytest.raises(RuntimeError):
        oracle.plan(pts, frq, +1, 1e-9, mode=2, max_grid_bytes=1024)


def test_config1_oracle_vs_reference_golden(oracle):
    # BASELINE configs[0] exactly (N = 1e4): the C restatement against the
    # reference's own apply / apply_adjoint on the reference's operator file
    from tests.conftest import config1_operator
    path, g = config1_operator()
    op = oracle.op(path)
    assert rel_l2(op.apply(g["f"]), g["q"]) <= 1e-12
    assert rel_l2(op.apply_adjoint(g["u"]), g["qa"]) <= 1e-12
