"""GPU parity of the device batch layer (csrc/kernels_batch.cuh) against the
CPU oracle's restatement of the reference batch kernels
(oracle.expand <- linalg.py:246-288, oracle.expm_clenshaw <-
chebyshev.py:259-306, numpy matmul <- linalg.py:204-233), complex128 and
complex64 (computed in complex64 arithmetic, as the reference does).

Gates: complex128 max-abs deviation <= 64 d u max(1, |G|) (+ the plan's
predicted truncation error for expm, which both sides share), complex64 the
same with u = 2^-24; the reference's own gemm-vs-naive tolerance is
8 d u mag + 32 u (test_linalg.py:120-134).
"""

import numpy as np
import pytest

from helpers import random_hermitian

import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu

U = {"fp64": 2.0 ** -53, "fp32": 2.0 ** -24}
BITS = {"fp64": 64, "fp32": 32}


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("d", [1, 2, 3, 4, 8, 13, 16, 17, 32, 33, 48, 64, 65, 96, 128, 200])
def test_expm_batch_against_oracle(d, precision):
    import oracle
    rng = np.random.default_rng(1000 + d)
    prec = sp.Precision.parse(precision)
    bound = 0.9 * sp.norm_capability(13, prec)
    count = 37 if d <= 64 else 5
    mats = np.stack([random_hermitian(rng, d, norm=bound * rng.uniform(0.3, 1.0))
                     for _ in range(count)])
    g = sp.MatrixBatch.from_matrices(mats, prec)
    plan = sp.make_plan(-bound, bound, prec)
    ws = sp.Workspace(d, prec)
    u = sp.expm_batch(g, plan, ws).to_array()
    ref = oracle.expm_clenshaw(g.to_array(), {
        "alpha": plan.alpha, "beta": plan.beta, "m_max": plan.m_max,
        "coeffs": plan.coeffs, "phase": plan.phase}, BITS[precision])
    tol = 64 * d * U[precision] * max(1.0, bound) + 10 * plan.predicted_error
    dev = np.abs(u - ref).max()
    assert u.dtype == prec.complex_dtype
    assert dev <= tol, (dev, tol)
    # workspace reuse: second call on the same workspace is identical
    again = sp.expm_batch(g, plan, ws).to_array()
    assert np.array_equal(again, u)


@pytest.mark.parametrize("center", [0.0, 1.5])
def test_expm_batch_asymmetric_interval(center):
    """Nonzero center exercises the shift and the scalar phase (d <= 64 fused
    and d > 64 multi-launch paths)."""
    rng = np.random.default_rng(7)
    for d in (3, 80):
        mats = np.stack([random_hermitian(rng, d, norm=0.8) + center * np.eye(d)
                         for _ in range(4)])
        plan = sp.make_plan(center - 1.0, center + 1.0, "fp64")
        u = sp.expm_batch(sp.MatrixBatch.from_matrices(mats), plan,
                          sp.Workspace(d, "fp64")).to_array()
        for k in range(4):
            w, v = np.linalg.eigh(mats[k])
            exact = (v * np.exp(-1j * w)) @ v.conj().T
            assert np.abs(u[k] - exact).max() <= 1e-12


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("d,n_terms,count", [(2, 3, 1000), (7, 4, 333), (64, 5, 50),
                                             (128, 3, 9)])
def test_expand_against_oracle(d, n_terms, count, precision):
    import oracle
    rng = np.random.default_rng(d * 31 + n_terms)
    terms = [random_hermitian(rng, d, norm=1.0) for _ in range(n_terms)]
    table = np.column_stack([np.ones(count), rng.uniform(-1, 1, (count, n_terms - 1))])
    got = sp.expand_linear_combination(terms, table, 0.37, precision).to_array()
    ref = oracle.expand(terms, table, 0.37, BITS[precision])
    assert got.dtype == ref.dtype
    assert np.abs(got - ref).max() <= 64 * U[precision] * n_terms


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("d,count", [(1, 7), (2, 100), (5, 33), (64, 4), (65, 3), (130, 2)])
@pytest.mark.parametrize("alpha,beta", [(1.0, 0.0), (2.0, -1.0), (0.5 - 0.25j, 1.0 + 2.0j)])
def test_gemm_strided_batched_against_numpy(d, count, alpha, beta, precision):
    rng = np.random.default_rng(d + count)
    mk = lambda: rng.standard_normal((count, d, d)) + 1j * rng.standard_normal((count, d, d))
    a, b, c0 = mk(), mk(), mk()
    prec = sp.Precision.parse(precision)
    A, B = sp.MatrixBatch.from_matrices(a, prec), sp.MatrixBatch.from_matrices(b, prec)
    C = sp.MatrixBatch.from_matrices(c0, prec)
    sp.gemm_strided_batched(A, B, alpha, beta, C)
    ref = alpha * np.matmul(A.to_array().astype(np.complex128), B.to_array().astype(np.complex128))
    if beta != 0:
        ref = ref + beta * c0.astype(prec.complex_dtype).astype(np.complex128)
    mag = np.abs(a).max() * np.abs(b).max() * d * abs(alpha) + abs(beta) * np.abs(c0).max()
    assert np.abs(C.to_array() - ref).max() <= 8 * d * U[precision] * mag + 32 * U[precision]


def test_build_exponent_batches_against_oracle():
    """build_exponent_batch (midpoint / simpson) and
    build_magnus_exponent_batch against the oracle's expansion tables."""
    import oracle
    rng = np.random.default_rng(99)
    d, n = 6, 3
    h0 = random_hermitian(rng, d, norm=1.0)
    hs = [random_hermitian(rng, d, norm=1.0) for _ in range(n)]
    values = rng.uniform(-1, 1, (41, n))
    system = sp.ControlSystem(h0, hs)
    amps = sp.ControlAmplitudes(values, 0.05)
    for mode in ("midpoint", "simpson", "magnus"):
        if mode == "magnus":
            g = sp.build_magnus_exponent_batch(sp.build_effective_system(system), amps)
        else:
            g = sp.build_exponent_batch(system, amps, mode)
        terms, *_ = oracle.effective_terms(h0, hs, mode == "magnus")
        table, scale, count = oracle.slice_table(values, 0.05, mode)
        ref = oracle.expand(terms, table, scale, 64)
        assert g.count == count
        assert np.abs(g.to_array() - ref).max() <= 1e-15, mode
