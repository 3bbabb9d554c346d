"""Host side of the Gauss-Legendre extension modes: sampling at the nodes,
weight tables (package vs oracle restatement), bounds, slice counts."""

import math

import numpy as np
import pytest

import oracle
import paper_2108_07126_b200 as sp
from paper_2108_07126_b200.magnus import build_effective_system, gauss_magnus_bound, gauss_table


def test_driven_qubit_samples_at_the_gauss_nodes():
    q = sp.DrivenQubit()
    amps = q.amplitudes(8, "gauss-legendre")
    dt = q.duration / 8
    assert amps.dt == dt
    t = np.array([(2 * k + 1 + s / math.sqrt(3.0)) * dt for k in range(4) for s in (-1, 1)])
    assert np.allclose(amps.values[:, 0], np.cos(t), rtol=0, atol=1e-15)
    assert np.allclose(amps.values[:, 1], np.sin(t), rtol=0, atol=1e-15)
    with pytest.raises(sp.SamplingParityError):
        q.amplitudes(7, "gauss-legendre")
    assert sp.coerce_pts(7, "gauss-legendre") == 8 and sp.coerce_pts(1, "gauss-legendre") == 2


@pytest.mark.parametrize("magnus", [False, True])
def test_weight_table_matches_the_oracle(magnus):
    rng = np.random.default_rng(3)
    values = rng.uniform(-1, 1, (40, 3))
    amps = sp.ControlAmplitudes(values, 0.07)
    table, scale = gauss_table(amps, magnus)
    ref, rscale, count = oracle.gauss_table(values, 0.07, magnus)
    assert count == 20 and scale == rscale == 0.14
    assert np.array_equal(table, ref)


def test_bound_and_slice_count():
    rng = np.random.default_rng(4)
    h = [0.5 * (a + a.conj().T) for a in
         (rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4)) for _ in range(3))]
    system = sp.ControlSystem(h[0], h[1:])
    eff = build_effective_system(system)
    dt = 0.01
    expect = (2 * dt * sum(system.norms)
              + 2 * math.sqrt(3) * dt * dt / 3 * (sum(eff.drift_comm_norms)
                                                 + sum(eff.cross_comm_norms)))
    assert math.isclose(gauss_magnus_bound(eff, dt), expect, rel_tol=1e-15)
    ctx = sp.create()
    ctx.set_hamiltonian(system, magnus=True, quadrature="gauss-legendre")
    assert ctx.mode == "gauss4"
    assert ctx.slice_count(10) == 5
    assert math.isclose(ctx.bound(dt), expect, rel_tol=1e-15)
    with pytest.raises(sp.SamplingParityError):
        ctx.slice_count(9)
    ctx.set_hamiltonian(system, quadrature="gauss-legendre")
    assert ctx.mode == "gauss2" and math.isclose(ctx.bound(dt), 2 * dt * sum(system.norms))
    ctx.close()
