"""Host schedule of the scaling-and-squaring extension (scaling.py): the
chosen (m, s) keeps nu / 2^s inside the order-m capability and minimises
(m + 1) + 2 s over the order grid."""

import math

import pytest

from paper_2108_07126_b200.chebyshev import ORDER_GRID, norm_capability
from paper_2108_07126_b200.linalg import Precision
from paper_2108_07126_b200.scaling import schedule


@pytest.mark.parametrize("precision", [Precision.FP64, Precision.FP32])
@pytest.mark.parametrize("nu", [0.01, 0.5, 4.0, 4.5, 20.0, 1e3, 1e6])
def test_schedule_is_feasible_and_minimal(nu, precision):
    m, s = schedule(nu, precision)
    assert nu / 2.0 ** s <= norm_capability(m, precision)
    cost = m + 1 + 2 * s
    for mm in ORDER_GRID:
        cap = norm_capability(mm, precision)
        ss = 0 if nu <= cap else math.ceil(math.log2(nu / cap))
        while nu / 2.0 ** ss > cap:
            ss += 1
        assert cost <= mm + 1 + 2 * ss


def test_schedule_respects_an_order_override():
    m, s = schedule(20.0, Precision.FP64, m_max=7)
    assert m == 7 and 20.0 / 2 ** s <= norm_capability(7, Precision.FP64)
