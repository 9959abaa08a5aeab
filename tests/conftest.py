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
