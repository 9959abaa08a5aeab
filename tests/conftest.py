"""Shared pytest configuration.

Markers: ``gpu`` -- needs a CUDA device (run on a B200 with ``-m gpu``);
everything else runs on CPU (``-m "not gpu"``).
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")


def golden_cases():
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)["cases"]


def golden(name):
    return os.path.join(GOLDEN, name + ".sbdop"), dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reflib():
    from oracle.oracle import REF_SO, RefLib
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref/libsbdref.so not built (needs /root/reference at build time)")
    return RefLib()


def config1_operator():
    """(path, golden arrays) of BASELINE configs[0] (N = 1e4 Laplace disk): the
    reference's own operator file, rebuilt by the reference's assemble
    (oracle/_ref) when absent and checked bit-for-bit against the SHA-256 the
    golden generator recorded (tests/golden/make_golden.py config1)."""
    import hashlib
    name = "cfg1_lap_disk_n10000"
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        meta = json.load(fh)["config1"]
    path = os.path.join(GOLDEN, name + ".sbdop")
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    if not os.path.exists(path):
        from oracle.oracle import REF_SO, RefLib
        if not os.path.exists(REF_SO):
            pytest.skip("config-1 operator needs oracle/_ref (the reference) to rebuild")
        ref = RefLib()
        tmp = path + f".{os.getpid()}.tmp"
        ref.assemble_save(tmp, g["points"], a_override=meta["a_override"])
        os.replace(tmp, path)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    assert sha == meta["sha256"], "rebuilt config-1 operator differs from the golden's"
    return path, g
