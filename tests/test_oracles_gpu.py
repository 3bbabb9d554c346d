"""GPU analytic oracles and state propagation.

``midpoint_reference`` (studies.py:123-153) runs on the device
(qubit_reference_kernel: exact per-slice SU(2) rotations, the su(2) lanes and
fused ordered tail); it is checked against the 80-bit host restatement of the
same recipe (oracle.midpoint_reference_ld) and, at the reference's 1e7 steps,
against the closed form through validate_analytic_oracle (studies.py:159-178).
``apply`` / ``apply_batch`` (propagator.py:105-118) run on the device and are
checked against numpy products.
"""

import numpy as np
import pytest

import oracle
import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("steps", [1, 2, 7, 1000, 100_000, 1_000_000])
def test_midpoint_reference_matches_80bit_recipe(steps):
    q = sp.DrivenQubit()
    u = sp.midpoint_reference(q, steps)
    ref = oracle.midpoint_reference_ld(q.w0, q.w1, q.wrf, q.duration, steps)
    err = float(np.abs(u - ref).max())
    # float64 rotations folded over `steps` slices: ~u * sqrt(steps) growth
    tol = 1e-14 * max(1.0, steps) ** 0.75
    print(f"\n[oracle] midpoint_reference steps={steps}: |gpu - 80-bit| {err:.3e} (tol {tol:.1e})")
    assert err <= tol
    assert abs(abs(np.linalg.det(u)) - 1.0) < 1e-14 * max(1.0, steps) ** 0.75


def test_midpoint_reference_edge_cases():
    assert np.array_equal(sp.midpoint_reference(sp.DrivenQubit(), 0), np.eye(2))
    assert np.array_equal(sp.midpoint_reference(sp.DrivenQubit(w0=0.0, w1=0.0), 100), np.eye(2))
    # a non-rotating field: one constant rotation per slice
    q = sp.DrivenQubit(w0=1.0, w1=0.3, wrf=0.0, duration=2.0)
    u = sp.midpoint_reference(q, 5000)
    assert np.abs(u - q.exact_propagator()).max() < 1e-12


def test_validate_analytic_oracle_at_the_reference_step_count():
    err = sp.validate_analytic_oracle(sp.DrivenQubit(), steps=10_000_000)
    print(f"\n[oracle] 1e7-step midpoint reference vs closed form: {err:.3e}")
    assert err <= 1e-8


def test_apply_vector_and_density():
    rng = np.random.default_rng(5)
    for d in (1, 2, 5, 32, 128):
        a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        u, _ = np.linalg.qr(a)
        psi = rng.standard_normal(d) + 1j * rng.standard_normal(d)
        rho = np.outer(psi, psi.conj())
        assert np.allclose(sp.apply(u, psi), u @ psi, rtol=0, atol=1e-13 * d)
        assert np.allclose(sp.apply(u, rho), u @ rho @ u.conj().T, rtol=0,
                           atol=1e-13 * d * np.abs(rho).max())


def test_apply_batch_and_dtypes():
    rng = np.random.default_rng(6)
    d, count = 16, 37
    u, _ = np.linalg.qr(rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d)))
    psis = rng.standard_normal((count, d)) + 1j * rng.standard_normal((count, d))
    out = sp.apply_batch(u, psis)
    assert out.dtype == np.complex128
    assert np.allclose(out, psis @ u.T, rtol=0, atol=1e-12)
    rhos = np.einsum("ki,kj->kij", psis, psis.conj())
    out = sp.apply_batch(u, rhos)
    assert np.allclose(out, u @ rhos @ u.conj().T, rtol=0, atol=1e-11)
    out32 = sp.apply_batch(u.astype(np.complex64), psis.astype(np.complex64))
    assert out32.dtype == np.complex64
    assert np.allclose(out32, psis @ u.T, rtol=0, atol=1e-4)


def test_apply_accepts_a_result_and_rejects_bad_shapes():
    with sp.create() as ctx:
        h0, hs = 0.5 * np.diag([1.0, -1.0]).astype(complex), [np.array([[0, 1], [1, 0]], complex)]
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        res = ctx.equiprop(sp.ControlAmplitudes(np.zeros((10, 1)), 0.1))
    psi = np.array([1.0, 0.0], dtype=complex)
    assert np.allclose(sp.apply(res, psi), res.u @ psi)
    with pytest.raises(sp.ShapeError):
        sp.apply(res, np.ones(3))
    with pytest.raises(sp.ShapeError):
        sp.apply(np.ones((2, 3)), psi)
