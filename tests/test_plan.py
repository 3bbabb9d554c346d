"""Host plan through the C ABI (csrc/plan.cpp) is bit-exact against the
reference's outputs (tests/golden/plan.npz) and keeps its error contract
(reference tests/test_chebyshev.py)."""

import math

import numpy as np
import pytest

import paper_2108_07126_b200 as sp

CAPABILITY_TABLE = {  # reference test_chebyshev.py:36-49 / test_acceptance.py:28-33
    3: ("0.033", "2e-04"), 5: ("0.219", "0.008"), 7: ("0.620", "0.050"),
    9: ("1.218", "0.163"), 11: ("1.980", "0.368"), 13: ("2.873", "0.677"),
    15: ("3.873", "1.088"), 17: ("4.959", "1.596"), 19: ("6.118", "2.194"),
    21: ("7.336", "2.874"), 23: ("8.606", "3.627"), 25: ("9.919", "4.447"),
}


def test_bessel_bitwise(plan_golden):
    g = plan_golden
    got = np.array([[sp.bessel_j(int(k), x) for x in g["bessel_x"]] for k in g["bessel_k"]])
    assert np.array_equal(got, g["bessel_j"])


def test_bessel_known_values():
    assert sp.bessel_j(0, 0.0) == 1.0
    assert sp.bessel_j(3, 0.0) == 0.0
    expect = 0.7651976865579666
    assert abs(sp.bessel_j(0, 1.0) - expect) <= 4 * np.spacing(expect)


@pytest.mark.parametrize("k,x", [(-1, 1.0), (65, 1.0), (2.5, 1.0), (0, -0.1), (0, 64.001),
                                 (0, math.nan)])
def test_bessel_domain_errors(k, x):
    with pytest.raises(sp.DomainError):
        sp.bessel_j(k, x)


def test_chebyshev_error_bitwise(plan_golden):
    g = plan_golden
    got = np.array([[sp.chebyshev_error(m, s) for s in g["err_spans"]] for m in sp.ORDER_GRID])
    assert np.array_equal(got, g["chebyshev_error"])


def test_capability_bitwise_and_table(plan_golden):
    got = np.array([[sp.norm_capability(m, p) for m in sp.ORDER_GRID] for p in ("fp32", "fp64")])
    assert np.array_equal(got, plan_golden["capability"])
    for m, (single, double) in CAPABILITY_TABLE.items():
        assert sp.format_capability(sp.norm_capability(m, "fp32")) == single
        assert sp.format_capability(sp.norm_capability(m, "fp64")) == double


def test_select_bitwise(plan_golden):
    g = plan_golden
    for pi, prec in enumerate(("fp32", "fp64")):
        for bi, b in enumerate(g["select_bounds"]):
            expect = int(g["select_m"][pi, bi])
            if expect < 0:
                with pytest.raises(sp.StepTooLargeError) as ei:
                    sp.select_m_max(b, prec)
                assert ei.value.capability == pytest.approx(sp.norm_capability(25, prec))
                assert ei.value.norm_bound == b
            else:
                assert sp.select_m_max(b, prec) == expect


def test_make_plan_bitwise(plan_golden):
    g = plan_golden
    for pi, prec in enumerate(("fp32", "fp64")):
        for bi, b in enumerate(g["plan_betas"]):
            if g["plan_m"][pi, bi] < 0:
                with pytest.raises(sp.StepTooLargeError):
                    sp.make_plan(-b, b, prec)
                continue
            plan = sp.make_plan(-b, b, prec)
            assert plan.m_max == g["plan_m"][pi, bi]
            assert np.array_equal(plan.coeffs, g["plan_coeffs"][pi, bi, :plan.m_max + 1])
            assert plan.predicted_error == g["plan_predicted_error"][pi, bi]
            assert plan.phase == 1.0


def test_plan_known_coefficients():
    # reference test_chebyshev.py:195-209
    plan = sp.make_plan(-1.0, 1.0, "fp64")
    assert plan.coeffs[0].real == pytest.approx(0.7651976865579666, rel=1e-15)
    assert plan.coeffs[1].imag == pytest.approx(-0.4400505857449335, rel=1e-15)
    assert sp.make_plan(-0.5, 0.5, "fp64").m_max == 13
    assert sp.make_plan(-0.05, 0.05, "fp64").m_max == 7


def test_plan_errors():
    with pytest.raises(sp.ConfigError):
        sp.make_plan(1.0, -1.0, "fp64")
    with pytest.raises(sp.ConfigError):
        sp.make_plan(-1.0, 1.0, "fp64", m_max=4)
    with pytest.raises(sp.StepTooLargeError):
        sp.make_plan(-50.0, 50.0, "fp64", m_max=3)
    with pytest.raises(sp.ConfigError):
        sp.make_plan(-1.0, 1.0, "fp16")
    with pytest.raises(sp.DomainError):
        sp.select_m_max(-1.0, "fp64")
    with pytest.raises(sp.ConfigError):
        sp.norm_capability(4, "fp64")
