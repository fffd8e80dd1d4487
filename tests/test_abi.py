"""The C-ABI library: loads, exports every declared symbol, and its host-only
logic (validation, shard plans, the random stream's libm check) — no GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1901_04200_b200 import configs, engine
from paper_1901_04200_b200.cabi import MarshalledModel
from paper_1901_04200_b200.model import load_model_spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lanetape_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ltg_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = engine.load_library()
    names = declared_symbols()
    assert len(names) >= 18
    for n in names:
        assert hasattr(lib, n), n


def test_abi_version():
    assert engine.load_library().ltg_abi_version() == 1


def test_rng_log_restatement_matches_host_libm():
    r = engine.rng_selftest(1 << 21)
    assert r["found"] and r["exact"] and r["mismatches"] == 0


@pytest.mark.parametrize("paths", [1, 127, 128, 1000, 1 << 20, (1 << 22) + 5, 1 << 26])
def test_shard_plan_partitions_paths(paths):
    for world in (1, 2, 3, 4, 8):
        plans = [engine.shard_plan(paths, r, world) for r in range(world)]
        cp = plans[0]["chunk_paths"]
        # chunk size depends on the total only: partials are rank-count independent
        assert all(p["chunk_paths"] == cp and p["n_chunks"] == plans[0]["n_chunks"] for p in plans)
        assert cp % 128 == 0
        assert plans[0]["n_chunks"] == -(-paths // cp)
        covered = 0
        for r, p in enumerate(plans):
            assert p["path_begin"] == covered
            covered = p["path_end"]
            # equal-sized (padded) rows so every rank's block sits at rank * per
            per = -(-p["n_chunks"] // world)
            assert p["chunk_begin"] == min(per * r, p["n_chunks"])
        assert covered == paths


def test_shard_plan_rejects_bad_arguments():
    with pytest.raises(ValueError):
        engine.shard_plan(0, 0, 1)
    with pytest.raises(ValueError):
        engine.shard_plan(10, 2, 2)


def test_model_validation_precedes_device_use(golden_dir):
    # std::invalid_argument sites of heston.hpp:199-299 -> LTG_EINVAL (ValueError)
    spec = load_model_spec(os.path.join(golden_dir, "heston_small.json"))
    spec.instruments[0].maturity_step = spec.mc.steps + 1
    with pytest.raises(ValueError, match="maturity_step"):
        engine.Engine(spec)
    spec = load_model_spec(os.path.join(golden_dir, "heston_small.json"))
    spec.grid.s_nodes = [100.0, 90.0, 115.0]
    with pytest.raises(ValueError, match="ascending"):
        engine.Engine(spec)
    spec = load_model_spec(os.path.join(golden_dir, "heston_small.json"))
    spec.heston.rho = 1.0
    with pytest.raises(ValueError, match="rho"):
        engine.Engine(spec)


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu(golden_dir):
    spec = load_model_spec(os.path.join(golden_dir, "heston_small.json"))
    with pytest.raises(engine.EngineError):
        engine.Engine(spec)
