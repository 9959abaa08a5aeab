"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs in the build container only (needs oracle/_ref/libsbdref.so, i.e. the
reference sources under /root/reference compiled by oracle/Makefile). The
outputs are committed so that the CPU oracle can be pinned -- and the GPU path
checked -- on machines where /root/reference does not exist.

    python tests/golden/make_golden.py

Each operator case writes <name>.sbdop (the reference's own SBDOPv1 file from
CompressedOperator::assemble + save) and <name>.npz holding the inputs f / u and
the reference's outputs of CompressedOperator::load(...).apply(f) and
.apply_adjoint(u) plus the intermediate spectrum NufftPlan(src, xi, -).apply(f).
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import RefLib  # noqa: E402

from tests.clouds import disk_cloud, square_cloud, star_curve_cloud  # noqa: E402


def case(ref, name, src, tgt=None, kind=0, k=0.0, eps=1e-6, a_override=0.0, f_complex=False,
         seed=0):
    path = os.path.join(HERE, name + ".sbdop")
    info = ref.assemble_save(path, src, tgt, kind=kind, k=k, eps=eps, a_override=a_override)
    rng = np.random.default_rng(seed)
    n_src = len(src)
    n_tgt = n_src if tgt is None else len(tgt)
    f = rng.standard_normal(n_src) + (1j * rng.standard_normal(n_src) if f_complex else 0.0)
    u = rng.standard_normal(n_tgt) + 1j * rng.standard_normal(n_tgt)
    op = ref.load(path)
    q = op.apply(f, n_tgt)
    qa = op.apply_adjoint(u, n_src)
    raw = ref.raw(path)
    spec = raw.stage(1, f, int(info["n_xi"]))
    np.savez_compressed(os.path.join(HERE, name + ".npz"), f=f, q=q, u=u, qa=qa, spectrum=spec)
    info.update(name=name, n_src=n_src, n_tgt=n_tgt, kind=kind, k=k, eps=eps,
                a_override=a_override)
    print(json.dumps(info))
    return info


CFG1 = "cfg1_lap_disk_n10000"


def config1(ref, path=None):
    """BASELINE.json configs[0] exactly: Laplace, N = 1e4 i.i.d. uniform in the
    disk of diameter 1, eps = 1e-6, delta_min = 2.74/sqrt(N), real f. The
    reference's operator file (7.8 MB) is not committed: the reference's own
    assemble rebuilds it bit-identically in ~1 s (tests/conftest.py
    config1_operator checks its SHA-256 against the manifest); the points, f,
    u and the reference's outputs are committed."""
    import hashlib
    rng = np.random.default_rng(10_000)
    src = disk_cloud(10_000, rng)
    d = ref.diameter(src)
    path = path or os.path.join(HERE, CFG1 + ".sbdop")
    a = (2.74 / np.sqrt(10_000)) / d
    info = ref.assemble_save(path, src, a_override=a)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    return src, a, info, sha


def config1_case(ref):
    src, a, info, sha = config1(ref)
    rng = np.random.default_rng(11)
    n = len(src)
    f = rng.standard_normal(n) + 0j
    u = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    path = os.path.join(HERE, CFG1 + ".sbdop")
    op = ref.load(path)
    q = op.apply(f, n)
    qa = op.apply_adjoint(u, n)
    np.savez_compressed(os.path.join(HERE, CFG1 + ".npz"), points=src, f=f, q=q, u=u, qa=qa)
    info.update(name=CFG1, n_src=n, n_tgt=n, kind=0, k=0.0, eps=1e-6, a_override=a, sha256=sha,
                committed_operator=False)
    print(json.dumps(info))
    return info


def nufft_kats(ref):
    rng = np.random.default_rng(17)
    out = {}
    pts = rng.uniform(-0.85, 0.85, (300, 2))
    frq = rng.uniform(-40.0, 40.0, (311, 2))
    c = rng.uniform(-1, 1, 300) + 1j * rng.uniform(-1, 1, 300)
    v = rng.uniform(-1, 1, 311) + 1j * rng.uniform(-1, 1, 311)
    arrays = dict(pts=pts, frq=frq, c=c, v=v)
    for tol in (1e-4, 1e-8, 1e-12):
        for sign in (-1, 1):
            a, meta = ref.nufft(pts, frq, c, sign, tol, mode=2)
            t, _ = ref.nufft(pts, frq, v, sign, tol, mode=2, transpose=True)
            key = f"tol{tol:.0e}_s{'p' if sign > 0 else 'm'}"
            arrays["apply_" + key] = a
            arrays["transpose_" + key] = t
            out[key] = meta
    d, _ = ref.nufft(pts, frq, c, +1, 1e-9, mode=1)
    arrays["direct_p"] = d
    xs = np.array([0.0, 1e-3, 0.5, 1.0, 3.7, 10.0, 18.85, 23.56, 25.918, 40.0])
    arrays["i0_x"] = xs
    arrays["i0"] = np.array([ref.bessel("i0", x) for x in xs])
    np.savez_compressed(os.path.join(HERE, "nufft_kat.npz"), **arrays)
    return out


def main():
    ref = RefLib()
    cases = []
    rng = np.random.default_rng(2026)
    # (1) config-1 shape, scaled to N=1000: Laplace, uniform disk of diameter 1,
    #     delta_min = 2.74/sqrt(N), real f ~ N(0,1) (BASELINE.json configs[0]).
    src = disk_cloud(1000, rng)
    d = ref.diameter(src)
    cases.append(case(ref, "lap_disk_n1000", src, a_override=(2.74 / np.sqrt(1000)) / d, seed=1))
    # (2) Helmholtz (config-3 shape), kappa = k * dmax = 2 pi * 5, complex f.
    src = disk_cloud(800, rng)
    d = ref.diameter(src)
    cases.append(case(ref, "helm_disk_n800", src, kind=1, k=2 * np.pi * 5 / d,
                      a_override=(2.74 / np.sqrt(800)) / d, f_complex=True, seed=2))
    # (3) BEM-like star curve (config-2 shape), reference a-rule, eps 1e-6.
    src = star_curve_cloud(1500, rng)
    cases.append(case(ref, "lap_star_n1500", src, seed=3))
    # (4) two clouds (non-single operator), overlapping squares, eps 1e-5.
    s = square_cloud(900, rng)
    t = square_cloud(800, rng) + np.array([0.4, 0.1])
    cases.append(case(ref, "lap_two_clouds", s, t, eps=1e-5, f_complex=True, seed=4))
    # (4b) two clouds where fwd_in is direct (50 * N_xi <= 2^20) and fwd_out fast.
    s = square_cloud(50, rng)
    t = square_cloud(1200, rng) + np.array([0.2, 0.3])
    cases.append(case(ref, "lap_mixed_paths", s, t, eps=1e-6, seed=7))
    # (5) tiny cloud: both plans take the exact direct path (N * N_xi <= 2^20).
    src = disk_cloud(60, rng)
    cases.append(case(ref, "lap_direct_n60", src, eps=1e-3, seed=5))
    # (6) Helmholtz, Robin regime (small k), two clouds far apart -> empty D.
    s = square_cloud(200, rng, side=0.8)
    t = square_cloud(150, rng, side=0.8) + np.array([2.5, 0.0])
    cases.append(case(ref, "helm_far_clouds", s, t, kind=1, k=0.3, eps=1e-4, f_complex=True,
                      seed=6))
    kat = nufft_kats(ref)
    cfg1 = config1_case(ref)
    with open(os.path.join(HERE, "manifest.json"), "w") as fh:
        json.dump({"cases": cases, "config1": cfg1, "nufft_kat": kat,
                   "generator": "tests/golden/make_golden.py via oracle/_ref/libsbdref.so"},
                  fh, indent=1)


if __name__ == "__main__":
    main()
