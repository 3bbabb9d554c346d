"""GPU parity of the u(2) lanes (kernels_su2.cuh on the 2 x 2 complex algebra).

d = 2 complex128 systems whose terms are bitwise Hermitian but not all
traceless (a random 2 x 2 system, a detuned qubit) run on the su(2) family's
lanes — TMA row stream for midpoint with 2 / 4 controls, the cp.async ring
otherwise — with two slices' complex Clenshaw pairs (Z = z0 I + Z') in
lockstep, 2 x 2 complex running products, the same ordered CTA tree and fused
tail.  complex64 keeps the reference's float32 sequence (lane_f32_kernel<2>).
Same gate as every other family: rel-Frobenius <= max(1e-12,
4 eps_self) against the oracle, over every mode, control counts 1..4, the
compiled (13) and runtime series orders, slice counts with odd tails and
partial last lanes, the sequential reduction and equiprop_all (lane mode), and
the amplitude-bound contract.
"""

import numpy as np
import pytest

from cases import random_inputs
from helpers import parity_tolerance, rel_fro

import oracle
import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu


def _gate(h0, hs, values, dt, mode, precision="fp64", reduction="pairwise", m_max=None,
          label=""):
    with sp.create(precision, m_max=m_max) as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        res = ctx.equiprop(sp.ControlAmplitudes(values, dt), reduction=reduction)
        kernel = ctx.last_timing()["kernel"]
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode, m_max=m_max,
                                    bits=32 if precision == "fp32" else 64)
    ref, ref_seq = oracle.reduce_pairwise(u), oracle.reduce_sequential(u)
    tol, eps_self = parity_tolerance(ref, ref_seq, precision)
    target = ref if reduction == "pairwise" else ref_seq
    err = rel_fro(res.u, target)
    print(f"\n[u2] {label} {mode} {precision} {reduction} slices={res.slice_count} "
          f"m={res.plan['m_max']} {kernel}: err {err:.3e} eps_self {eps_self:.3e} "
          f"tol {tol:.3e}")
    assert res.slice_count == u.shape[0]
    assert err <= tol
    return kernel


@pytest.mark.parametrize("mode", ["midpoint", "simpson", "magnus"])
@pytest.mark.parametrize("n_ctrl", [1, 2, 3, 4])
def test_random_u2_systems_every_mode(mode, n_ctrl):
    slices = 3001
    pts = slices if mode == "midpoint" else 2 * slices + 1
    h0, hs, values, dt = random_inputs(2, n_ctrl, pts, 500 + n_ctrl)
    kernel = _gate(h0, hs, values, dt, mode, label=f"N={n_ctrl}")
    assert kernel == "lane_u2_kernel"


@pytest.mark.parametrize("n_ctrl", [2, 4])
def test_complex64_keeps_the_reference_float32_sequence(n_ctrl):
    h0, hs, values, dt = random_inputs(2, n_ctrl, 4001, 600 + n_ctrl)
    kernel = _gate(h0, hs, values, dt, "midpoint", precision="fp32", label=f"N={n_ctrl}")
    assert kernel == "lane_f32_kernel<2>"


@pytest.mark.parametrize("beta", [1e-3, 0.05, 0.5, 2.0, 4.4])
@pytest.mark.parametrize("n_ctrl", [2, 4])
def test_series_orders(beta, n_ctrl):
    """beta spans the plan orders (7 and 13 compiled in for the TMA lanes,
    the rest at run time)."""
    h0, hs, values, dt = random_inputs(2, n_ctrl, 20000, 41, beta=beta)
    _gate(h0, hs, values, dt, "midpoint", label=f"beta={beta} N={n_ctrl}")


@pytest.mark.parametrize("n_ctrl", [1, 2])
@pytest.mark.parametrize("slices", [1, 2, 7, 33, 1001, 75777, 300001])
def test_slice_counts(slices, n_ctrl):
    """1 (one lane) .. more slices than lanes x round size (partial last lane
    on direct loads, short warps, odd pair tails)."""
    h0, hs, values, dt = random_inputs(2, n_ctrl, slices, 9)
    _gate(h0, hs, values, dt, "midpoint", label=f"slices N={n_ctrl}")


@pytest.mark.parametrize("mode,n_ctrl", [("midpoint", 2), ("midpoint", 3), ("simpson", 2),
                                         ("magnus", 4)])
def test_sequential_and_cumulative(mode, n_ctrl):
    """Lane mode: the sequential total and every cumulative propagator."""
    slices = 5001
    pts = slices if mode == "midpoint" else 2 * slices + 1
    h0, hs, values, dt = random_inputs(2, n_ctrl, pts, 71)
    kernel = _gate(h0, hs, values, dt, mode, reduction="sequential", label="sequential")
    assert kernel == "lane_u2_kernel"
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        cum = ctx.equiprop_all(sp.ControlAmplitudes(values, dt))
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode)
    ref_all = oracle.cumulative(u)
    err = max(rel_fro(cum.u_all[k], ref_all[k]) for k in (0, 1, slices // 2, slices - 1))
    print(f"\n[u2] equiprop_all {mode}: max err {err:.3e}")
    assert err <= 1e-12


def test_amplitude_bound_first_offender():
    import torch
    h0, hs, values, dt = random_inputs(2, 2, 40000, 13)
    values = values.copy()
    values[23456, 1] = 1.5
    values[30000, 0] = np.nan
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        d = torch.from_numpy(values).cuda()
        out = torch.empty((2, 2), dtype=torch.complex128, device="cuda")
        ctx.equiprop_device_ptr(d.data_ptr(), values.shape[0], 2, dt, out.data_ptr())
        torch.cuda.synchronize()
        assert ctx.last_timing()["kernel"] == "lane_u2_kernel"
        assert ctx.amplitude_violation() == 23456 * 2 + 1


def test_matches_the_complex_pair_kernel():
    """The u(2) lanes and lane_small_kernel<2,1> (SP_U2=0, in a subprocess)
    compute the same per-slice U; the totals agree to rounding."""
    import os
    import subprocess
    import sys
    import tempfile
    code = ("import numpy as np, sys; sys.path[:0] = ['tests/golden', '.'];"
            "from cases import random_inputs; import paper_2108_07126_b200 as sp;"
            "h0, hs, v, dt = random_inputs(2, 2, 60000, 5); ctx = sp.create();"
            "ctx.set_hamiltonian(sp.ControlSystem(h0, hs));"
            "u = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u;"
            "print(ctx.last_timing()['kernel']); np.save(sys.argv[1], u)")
    out = os.path.join(tempfile.mkdtemp(), "u.npy")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code, out], env=dict(os.environ, SP_U2="0"),
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().startswith("lane_small_kernel")
    h0, hs, values, dt = random_inputs(2, 2, 60000, 5)
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        u = ctx.equiprop(sp.ControlAmplitudes(values, dt)).u
        assert ctx.last_timing()["kernel"] == "lane_u2_kernel"
    assert rel_fro(u, np.load(out)) <= 1e-12
