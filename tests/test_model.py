"""Host-side model layer: JSON I/O, packing, validation, BASELINE configs."""
import json
import os

import pytest

from paper_1901_04200_b200 import configs
from paper_1901_04200_b200.model import (GradientReport, load_model_spec, model_spec_from_json,
                                         pack_params, to_json, unpack_params)


@pytest.mark.parametrize("name", ["heston_small", "heston_bs", "heston_calibrate",
                                  "heston_bench"])
def test_reference_configs_round_trip(golden_dir, name):
    s = load_model_spec(os.path.join(golden_dir, f"{name}.json"))
    assert model_spec_from_json(json.loads(json.dumps(to_json(s)))) == s
    assert list(to_json(s).keys()) == ["heston", "grid", "instruments", "mc"]


def test_pack_unpack(golden_dir):
    s = load_model_spec(os.path.join(golden_dir, "heston_small.json"))
    x = pack_params(s.heston, s.grid)
    assert len(x) == 5 + 9 and x[:5] == [1.5, 0.04, 0.5, -0.6, 0.09]
    x[0] = 3.0
    unpack_params(x, s.heston, s.grid)
    assert s.heston.kappa == 3.0
    with pytest.raises(ValueError):
        unpack_params(x[:-1], s.heston, s.grid)


def test_validation_messages(golden_dir):
    j = json.load(open(os.path.join(golden_dir, "heston_small.json")))
    j["instruments"][0]["kind"] = "digital"
    with pytest.raises(ValueError, match="kind"):
        model_spec_from_json(j)
    j = json.load(open(os.path.join(golden_dir, "heston_small.json")))
    j["mc"]["paths"] = 0
    with pytest.raises(ValueError, match="paths"):
        model_spec_from_json(j)


def test_report_json_key_order():
    r = GradientReport(1.0, [1.0], [0.5], [0.1, 0.2], 10, "recompute", 42)
    assert list(json.loads(r.to_json()).keys()) == ["G", "means", "lambda", "grad", "paths",
                                                    "mode", "seed"]


def test_baseline_config_shapes():
    c1, c2, c3, c4, c5 = (configs.ALL[k]() for k in ("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"))
    assert (c1.M, c1.m, c1.paths, c1.spec.mc.steps) == (9, 8, 1 << 16, 16)
    assert [c1.spec.instruments[i].maturity_step for i in range(8)] == [4, 4, 4, 8, 8, 16, 16, 16]
    assert (c2.M, c2.m, c2.paths, c2.spec.mc.steps) == (45, 40, 1 << 20, 64)
    assert all(0.15 <= v <= 0.35 for v in c2.truth[5:])
    assert (c3.M, c3.m, c3.paths, c3.spec.mc.steps) == (6, 60, 1 << 20, 756)
    assert c3.x[:5] == [2.0, 0.05, 0.4, -0.5, 0.05] and c3.truth[:5] == [1.5, 0.04, 0.5, -0.7, 0.04]
    assert (c4.M, c4.m, c4.paths, c4.spec.steps) == (16, 48, 1 << 22, 50)
    assert all(0.15 <= v <= 0.4 for v in c4.truth)
    assert c5.paths == 1 << 26 and c5.spec.mc.steps == 756
    # cfg1 targets: undiscounted Black-Scholes under the true piecewise vol
    assert len(c1.targets) == 8 and all(t > 0 for t in c1.targets)


def test_basket_correlation_is_spd():
    import numpy as np
    c = configs.cfg4()
    L = np.array(c.spec.chol).reshape(16, 16)
    corr = L @ L.T
    assert np.allclose(np.diag(corr), 1.0, atol=1e-14)
    assert np.allclose(L, np.tril(L))
    assert np.all(np.linalg.eigvalsh(corr) > 0)


def test_committed_targets_present():
    for name in ("cfg2", "cfg3"):
        c = configs.ALL[name]()
        t = configs.load_targets(c)
        assert t is not None and len(t) == c.m
