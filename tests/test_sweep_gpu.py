"""Detector curves (paper Fig. 8/10; reference threshold_sweep, src/campaign.cpp:299-357) on the GPU
through the C++ drop-in (tools/sweep_gpu: efta_b200::calibrate_thresholds + threshold_sweep on the
fault-tap build of the pair kernel) against the reference itself (oracle/_ref) with the same
calibration and trial seeds — the same random plans. Each backend calibrates its own base
thresholds (the reference procedure, per backend); the curves over the 10 log-spaced multipliers
must agree: identical false-alarm rates and detection rates within 0.1."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_detector_curves_match_reference():
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "tools"), "-s"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libefta_ref.so")):
        pytest.fail("oracle/_ref/libefta_ref.so missing")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sweep_compare.py"), "--n", "512", "--d", "64",
                          "--trials", "40", "--cal-trials", "40"], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr
    res = json.loads(out.stdout)
    assert "points" in res["gpu"], res["gpu"]
    g, ref = res["gpu"]["points"], res["reference"]["points"]
    assert len(g) == len(ref) == 10
    for (mg, dg, fg), (mr, dr, fr) in zip(g, ref):
        assert abs(mg - mr) < 1e-5 * mr  # printed with 6 significant digits
        assert fg == fr, (mg, fg, fr)
        assert abs(dg - dr) <= 0.1, (mg, dg, dr)
    # monotone: looser thresholds never raise either rate (reference acceptance check 10)
    for a, b in zip(g, g[1:]):
        assert a[1] >= b[1] and a[2] >= b[2]
