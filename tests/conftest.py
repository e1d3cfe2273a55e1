"""Shared pytest configuration.

Markers: ``gpu`` -- needs a B200 (run with ``-m gpu`` on the GPU box).  Everything
else runs on the CPU-only build container in a few minutes.
"""
import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA (B200) device")


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.bind import Reference, available
    if not available("ref"):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Reference()


@pytest.fixture(scope="session")
def hm():
    import paper_1708_09707_b200 as hm
    return hm


@pytest.fixture(scope="session")
def gpu(hm):
    if hm.device_count() < 1:
        pytest.fail("-m gpu test but no CUDA device is visible")
    return hm
