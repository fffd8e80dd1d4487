"""bench.py's engine arm on the GPU: the JSON line the driver reads (keys,
units, the roofline / cpu_baseline / e2e / clocks objects), on a small config
so the check takes seconds."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    return lines[0]


def test_engine_arm_json_contract():
    d = _run("--config", "cfg3", "--paths", "65536", "--steps", "2", "--warmup", "3",
             "--cpu-seconds", "0.5")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "clocks", "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["metric"] == "grad_G_mc_paths_per_sec" and d["unit"] == "paths/s"
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 2 and d["warmup"] == 3
    assert d["dtype"] == "f64" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "cfg3_heston"
    # per gradient_of_G: pass 1 + its two reduction kernels, and pass 2, whose
    # small table (2^16 paths x M = 6) its own last CTA reduces (fused_tail)
    assert d["gpu_launches"] == 2 * 4
    e = d["e2e"]
    assert e["unit"] == "paths/s" and 0 < e["value"] and e["h2d_bytes_per_step"] > 0
    r = d["roofline"]
    assert r["bound"] == "fp64" and 0 < r["frac"] < 1.2 and r["peak"] > 1.0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    # the census fractions, and SURVEY §8(d)'s W beside them (labelled, not the frac)
    assert 0 < r["frac"] <= r["executed_frac"] and r["survey_8d"]["W_per_path"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["clocks"]["samples"] >= 0
    assert "tangent" in d["alt_methods"]


def test_engine_arm_fp32_and_tangent_method():
    d = _run("--config", "cfg3", "--paths", "65536", "--steps", "1", "--warmup", "3",
             "--no-cpu-baseline", "--precision", "fp32", "--no-alt-method")
    assert d["dtype"] == "f32" and d["value"] > 0 and "alt_methods" not in d
    assert d["roofline"]["bound"] == "fp32" and 0 < d["roofline"]["frac"] < 1.2
    t = _run("--config", "cfg3", "--paths", "65536", "--steps", "1", "--warmup", "3",
             "--no-cpu-baseline", "--method", "tangent")
    assert t["method"] == "tangent" and t["value"] > 0


def test_gpus_n_drives_n_devices_loopback():
    # `bench.py --gpus N` without torchrun opens one context per device
    # (ltg_create_*_devices). With LTG_LOOPBACK=1 the N members share GPU 0
    # and exchange their chunk rows with device copies where NCCL would
    # all-gather: the report is bitwise the one-GPU report and n_gpus == N
    args = ["--config", "cfg3", "--paths", "50017", "--steps", "1", "--warmup", "3",
            "--no-cpu-baseline", "--no-alt-method"]
    one = _run("--gpus", "1", *args)
    env = dict(os.environ, LTG_LOOPBACK="1")
    for n in (2, 3):
        r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n),
                            *args], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
        assert r.returncode == 0, r.stderr[-3000:]
        (d,) = [json.loads(l) for l in r.stdout.splitlines() if l.strip().startswith("{")]
        assert d["n_gpus"] == n and "loopback" in d["config"]
        assert d["report_sha1"] == one["report_sha1"] and d["G"] == one["G"]
        assert d["value"] > 0


def test_gpus_n_fails_loudly_without_the_devices():
    # more devices than the machine has: the run must fail, not time fewer GPUs
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64",
                        "--config", "cfg1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode != 0 and "cannot open devices" in r.stderr
