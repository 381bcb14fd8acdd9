import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C ABI on cuda:0)")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cpuref():
    from oracle.cpu_ref import CpuRef
    return CpuRef()


@pytest.fixture(scope="session")
def reflib():
    from oracle.cpu_ref import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref/libqsync_ref.so not built (reference tree absent)")
    return RefLib()
