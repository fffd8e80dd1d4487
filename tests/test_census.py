"""The roofline numerator (census.py): algorithmic = executed minus the
redundant AS241 central-branch evaluations, weighted by the draw-store share."""
import pytest

from paper_1901_04200_b200 import census


def test_redundant_work_of_cfg3():
    # 15% of 1512 draws per RNG pass waste one 39-instruction central branch;
    # pass 1's last 4-step batch pads 8 slots of its 16-slot central batch
    # (pass 2 evaluates 8 slots per iteration: no padding)
    assert census.redundant("cfg3_heston", "fp64", "pass1") == \
        pytest.approx(0.15 * 1512 * 39 + 8 * 39)
    assert census.redundant("cfg5_heston_scaling", "fp64", "pass2_regen") == \
        pytest.approx(0.15 * 1512 * 39)
    assert census.redundant("cfg3_heston", "fp64", "pass2_store") == 0.0
    assert census.redundant("cfg4_basket16", "fp64", "pass2_regen") == 0.0


@pytest.mark.parametrize("name,prec", [("cfg1_gbm", "fp64"), ("cfg2_localvol", "fp64"),
                                       ("cfg3_heston", "fp64"), ("cfg3_heston", "fp32"),
                                       ("cfg4_basket16", "fp64"), ("cfg5_heston_scaling", "fp64")])
def test_algorithmic_below_executed_and_store_weighting(name, prec):
    for k in ("pass1", "pass2"):
        for f in (0.0, 0.3, 1.0):
            a = census.per_path(name, prec, k, f, "algorithmic")
            e = census.per_path(name, prec, k, f, "executed")
            assert 0 < a <= e
    # pass 2 reading stored draws does strictly less work (the basket's
    # epilogue draws nothing either way)
    r = census.per_path(name, prec, "pass2", 0.0)
    s = census.per_path(name, prec, "pass2", 1.0)
    assert s < r or name.startswith("cfg4")
    mid = census.per_path(name, prec, "pass2", 0.25)
    assert mid == pytest.approx(0.75 * r + 0.25 * s)


def test_survey_w_cross_check_figure():
    # SURVEY §8(d)'s preliminary W (bench.py roofline.survey_8d): an upper
    # figure beside the census, never below the executed count of both passes
    assert census.survey_w("cfg5_heston_scaling") == census.survey_w("cfg3_heston") == 2.6e5
    for name in ("cfg1_gbm", "cfg2_localvol", "cfg3_heston", "cfg4_basket16"):
        both = sum(census.per_path(name, "fp64", k, 0.0, "executed") for k in ("pass1", "pass2"))
        assert census.survey_w(name) >= both * 0.45  # the same order of magnitude
    assert census.survey_w("no_such_config") is None
