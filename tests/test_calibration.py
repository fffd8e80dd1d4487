"""The reference's calibrator, unchanged, on the GPU gradient:
acceptance criterion 7 (tests/acceptance.cpp:337-394) — gradient descent on
synthetic targets recovers kappa and theta within 1% from a 50% offset."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "examples", "calibrate_gpu")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="examples/calibrate_gpu not built")
def test_reference_calibrator_recovers_truth_on_gpu(golden_dir):
    out = subprocess.run([BIN, os.path.join(golden_dir, "heston_calibrate.json")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["converged"], r
    assert r["G"] <= 1e-10 * r["G0"]
    assert r["kappa_err"] <= 1e-2 and r["theta_err"] <= 1e-2, r
    # the calibrator's evaluations and their wall time are reported
    assert r["gradient_calls"] >= r["iters"] and r["value_calls"] >= 0
    assert 0 < r["ms_per_evaluation"] and r["calibration_seconds"] <= r["seconds"]
