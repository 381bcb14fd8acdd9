"""The quantizers' division-free rounding (csrc/common.cuh quant_rne / QScale) is
bit-identical to the oracle's IEEE division sat(rint(x / s)) (oracle/cpu_ref.c):
exhaustive over every float x with |x / s| in [1/4, 256] (outside, both give 0
or saturate) for edge scales (significand 1.0, 1 + ulp, all ones, the fast-path
limits) and seeded random ones.  CPU: the same IEEE single ops (x86 FMA)."""
import os
import subprocess

import numpy as np

from conftest import ROOT


def test_reciprocal_fma_rounding_is_exact(tmp_path):
    exe = str(tmp_path / "recip_check")
    subprocess.run(["gcc", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp", "-o", exe,
                    os.path.join(ROOT, "tests", "cpp", "recip_check.c"), "-lm"], check=True)
    edge = ["3f800000", "3f800001", "3f7fffff", "3c010204", "3d7fffff", "3bffffff",
            "12800000", "12ffffff", "71800000", "717fffff"]  # 2^-90 .. 2^100 ends
    rng = np.random.default_rng(11)
    e = rng.integers(-90, 100, 14)
    m = rng.integers(0, 1 << 23, 14)
    rand = ["%08x" % (((127 + int(a)) << 23) | int(b)) for a, b in zip(e, m)]
    r = subprocess.run([exe] + edge + rand, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout
    assert "mismatches 0" in r.stdout
    # the grid-float rounding (clamp + 1.5*2^23 add) vs sat(rint(v)) over all non-NaN quotients
    r = subprocess.run([exe, "grid"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout
    assert "checked 4278190082 mismatches 0" in r.stdout
