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
    assert engine.load_library().ltg_abi_version() == 3


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
    # std::invalid_argument sites of heston.hpp:30-130 -> LTG_EINVAL (ValueError)
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


def test_header_is_plain_c(tmp_path):
    # the drop-in boundary must be consumable from C (cgo / ctypes / JNI shims):
    # compile a translation unit that uses every declared type with gcc -std=c11
    import subprocess
    src = tmp_path / "use_abi.c"
    src.write_text('#include "lanetape_b200.h"\n'
                   "int main(void) {\n"
                   "  ltg_heston_model h = {0}; ltg_basket_model b = {0}; ltg_mc_config c = {0};\n"
                   "  ltg_report r = {0}; ltg_timing t = {0}; ltg_shard s = {0};\n"
                   "  (void)h; (void)b; (void)c; (void)r; (void)t; (void)s;\n"
                   "  return ltg_abi_version() == LTG_ABI_VERSION ? 0 : 1;\n}\n")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-fsyntax-only",
                        "-I", os.path.join(ROOT, "include"), str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_draws_entry_points_reject_missing_context_and_source():
    # ltg_gradient_of_G_draws / ltg_estimate_means_draws validate before any
    # device work: no context or no draw source -> LTG_EINVAL (no GPU needed)
    import ctypes as C
    from paper_1901_04200_b200.cabi import LTG_EINVAL, DrawsC, MCConfigC, ReportC
    L = engine.load_library()
    x = (C.c_double * 6)()
    t = (C.c_double * 60)()
    z = (C.c_double * 8)()
    d = DrawsC(C.cast(z, C.POINTER(C.c_double)), 1, 8)
    cfg = MCConfigC(1, 0, 0, 0, 0, 0)
    rep = ReportC()
    dp = C.POINTER(C.c_double)
    assert L.ltg_gradient_of_G_draws(None, C.cast(x, dp), 6, C.cast(t, dp), 60, C.byref(d),
                                     C.byref(cfg), C.byref(rep)) == LTG_EINVAL
    assert L.ltg_gradient_of_G_draws(None, C.cast(x, dp), 6, C.cast(t, dp), 60, None,
                                     C.byref(cfg), C.byref(rep)) == LTG_EINVAL
    assert L.ltg_estimate_means_draws(None, C.cast(x, dp), 6, C.byref(d), 1, C.cast(t, dp),
                                      None) == LTG_EINVAL
    assert L.ltg_estimate_means_draws(None, C.cast(x, dp), 6, None, 1, C.cast(t, dp),
                                      None) == LTG_EINVAL
