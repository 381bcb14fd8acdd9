"""Build the C++ drop-in check (tests/cpp/test_dropin.cpp) against
include/qsync_b200.hpp + libqsync_b200.so and run it on the GPU."""
import os
import subprocess

import pytest

from conftest import ROOT

CUDA = "/usr/local/cuda"


def _build(tmp_path):
    exe = str(tmp_path / "test_dropin")
    lib = os.path.join(ROOT, "paper_2407_02327_b200")
    cmd = ["g++", "-O2", "-std=c++17", os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp"),
           "-I" + os.path.join(ROOT, "include"), "-I" + f"{CUDA}/include", "-L" + lib,
           "-l:libqsync_b200.so", f"-Wl,-rpath,{lib}", "-L" + f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{CUDA}/lib64", "-o", exe]
    subprocess.run(cmd, check=True)
    return exe


def test_dropin_compiles(tmp_path):
    """CPU-side: the C++ mirror compiles and links against the C ABI."""
    _build(tmp_path)


@pytest.mark.gpu
def test_dropin_reference_sr_cases_and_acceptance_1_3(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASS" in r.stdout
