"""Gauss-Legendre Magnus modes on the device (north-star extension N2).

quadrature="gauss-legendre": two amplitude samples per slice of length 2 dt, at the
Gauss-Legendre nodes.  With magnus=True the exponent is the 4th-order
Gauss-Legendre Magnus step G = h (H(a) + H(b))/2 + (sqrt(3) h^2/12) i[H(a),
H(b)] over the reference's effective terms (magnus.py:36-85); magnus=False
keeps the node average (2nd order).  The reference has no such mode, so the
oracle rows are "parity unpinned" (oracle.gauss_table restates the formula);
the gates are (1) rel-Frobenius vs that oracle <= max(1e-12, 4 eps_self)
(1e-5 complex64) for every kernel family, and (2) the fitted convergence
orders on the driven qubit against its closed form (4 and 2).
"""

import numpy as np
import pytest

from cases import random_inputs
from helpers import parity_tolerance, rel_fro

import oracle
import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu


def _run(d, n_ctrl, slices, mode, precision="fp64", seed=1):
    h0, hs, values, dt = random_inputs(d, n_ctrl, 2 * slices, seed + d)
    dt = dt / 2.0  # a slice spans 2 dt
    with sp.create(precision) as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "gauss4",
                            quadrature="gauss-legendre")
        amps = sp.ControlAmplitudes(values, dt)
        res = ctx.equiprop(amps)
        kernel = ctx.last_timing()["kernel"]
    bits = 32 if precision == "fp32" else 64
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode, bits=bits)
    ref, seq = oracle.reduce_pairwise(u), oracle.reduce_sequential(u)
    tol, eps = parity_tolerance(ref, seq, precision)
    err = rel_fro(res.u, ref)
    print(f"\n[gauss] {mode} d={d} N={n_ctrl} slices={res.slice_count} {precision} {kernel} "
          f"m={res.plan['m_max']}: err {err:.3e} eps_self {eps:.3e} tol {tol:.3e}")
    assert res.slice_count == slices
    assert err <= tol
    return res


@pytest.mark.parametrize("mode", ["gauss2", "gauss4"])
@pytest.mark.parametrize("d", [2, 3, 8, 16, 32, 64, 128])
def test_every_family_matches_the_oracle(mode, d):
    _run(d, 2, 4000 if d <= 32 else (600 if d == 64 else 300), mode)


@pytest.mark.parametrize("d", [2, 8, 16])
def test_complex64(d):
    _run(d, 2, 300, "gauss4", precision="fp32")


def test_three_controls_cross_commutators():
    _run(8, 3, 1500, "gauss4")


def test_convergence_orders_on_the_driven_qubit():
    q = sp.DrivenQubit()
    pts = [16, 32, 64, 128, 256, 512, 1024]
    rows4 = sp.convergence_sweep(q, pts, magnus=True, quadrature="gauss-legendre")
    rows2 = sp.convergence_sweep(q, pts, magnus=False, quadrature="gauss-legendre")
    rowsm = sp.convergence_sweep(q, [p + 1 for p in pts], magnus=True)  # reference magnus
    o4, _ = sp.fit_convergence_order([p for p, _ in rows4], [e for _, e in rows4])
    o2, _ = sp.fit_convergence_order([p for p, _ in rows2], [e for _, e in rows2])
    print(f"\n[gauss] fitted orders: gauss4 {o4:.3f}, gauss2 {o2:.3f}")
    for (p, e4), (_, em) in zip(rows4, rowsm):
        print(f"  pts {p}: GL4 {e4:.3e}  reference magnus (pts+1) {em:.3e}")
    assert 3.8 <= o4 <= 4.3
    assert 1.9 <= o2 <= 2.1


def test_cumulative_and_sampling_parity():
    h0, hs, values, dt = random_inputs(8, 2, 2 * 300, 5)
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=True, quadrature="gauss-legendre")
        cum = ctx.equiprop_all(sp.ControlAmplitudes(values, dt / 2))
        with pytest.raises(sp.SamplingParityError, match="even number"):
            ctx.equiprop(sp.ControlAmplitudes(values[:-1], dt / 2))
    u, _ = oracle.slice_propagators(h0, hs, values, dt / 2, mode="gauss4")
    ref = oracle.cumulative(u)
    err = max(rel_fro(a, b) for a, b in zip(cum.u_all, ref))
    print(f"\n[gauss] cumulative: max rel err {err:.3e}")
    assert err <= 1e-12
