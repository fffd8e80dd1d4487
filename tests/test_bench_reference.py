"""bench.py's reference arm (CPU only: the reference's own gradient_of_G,
oracle/_ref) — its JSON contract, alone and under torchrun with two ranks
(rank 0 reports, the other rank exits 0 without work)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ref_or_skip():
    from oracle.bindings import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built and /root/reference absent")


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.strip().startswith("{")]


ARGS = ["--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1",
        "--ref-seconds", "0.2"]


def test_reference_arm_json_line():
    _ref_or_skip()
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + ARGS, cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    (line,) = _lines(r.stdout)
    assert line["impl"] == "reference" and line["metric"] == "grad_G_mc_paths_per_sec"
    assert line["unit"] == "paths/s" and line["value"] > 0 and line["higher_is_better"]
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": "paths/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"] == "cfg1_gbm" and line["steps"] == 2


def test_reference_arm_under_torchrun():
    _ref_or_skip()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29517",
           os.path.join(ROOT, "bench.py"), "--gpus", "2"] + ARGS
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_gpus_must_match_world_size():
    # under torchrun the job's GPU count is WORLD_SIZE; a different --gpus is
    # an error before any work (no silent single-GPU timing)
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2"] + ARGS,
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=3" in r.stderr
