"""GPU parity of the su(2) family (kernels_su2.cuh, lane_su2_kernel).

d = 2 systems whose terms are bitwise Hermitian and traceless (the paper's
driven qubit, any su(2) drive) run as quaternions: real Clenshaw pairs and
4-double running products.  These tests hold it to the same gate as every
other family (rel-Frobenius <= max(1e-12, 4 eps_self)
against the oracle, the bit-exact restatement of the reference), over every
mode, control count 1..4, the compiled series orders (3, 5, 7) and the
runtime order path (up to the m = 25 capability edge), slice counts from 1
(one lane) to 1e6 (the north-star size), plus the amplitude-bound contract
(first offender in row-major order, reference message) and the 80-bit
analytic gate of the driven qubit at 1e6 slices.
"""

import numpy as np
import pytest

from cases import qubit_inputs
from helpers import parity_tolerance, rel_fro

import oracle
import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu

SX = np.array([[0, 1], [1, 0]], dtype=complex)
SY = np.array([[0, -1j], [1j, 0]], dtype=complex)
SZ = np.array([[1, 0], [0, -1]], dtype=complex)


def traceless_terms(n_ctrl, seed):
    """Random traceless Hermitian 2 x 2 terms (real Pauli combinations)."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n_ctrl + 1):
        a = rng.standard_normal(3)
        out.append(a[0] * SX + a[1] * SY + a[2] * SZ)
    return out[0], out[1:]


def _run(h0, hs, values, dt, mode, m_max=None):
    with sp.create(m_max=m_max) as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        res = ctx.equiprop(sp.ControlAmplitudes(values, dt))
        return res, ctx.last_timing()["kernel"]


def _gate(h0, hs, values, dt, mode, m_max=None, label=""):
    res, kernel = _run(h0, hs, values, dt, mode, m_max)
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode, m_max=m_max)
    ref, ref_seq = oracle.reduce_pairwise(u), oracle.reduce_sequential(u)
    tol, eps_self = parity_tolerance(ref, ref_seq, "fp64")
    err = rel_fro(res.u, ref)
    print(f"\n[su2] {label} {mode} slices={res.slice_count} m={res.plan['m_max']} {kernel}: "
          f"err {err:.3e} eps_self {eps_self:.3e} tol {tol:.3e}")
    assert kernel == "lane_su2_kernel"
    assert res.slice_count == u.shape[0]
    assert err <= tol
    return res


@pytest.mark.parametrize("mode", ["midpoint", "simpson", "magnus"])
@pytest.mark.parametrize("n_ctrl", [1, 2, 3, 4])
def test_random_su2_systems_every_mode(mode, n_ctrl):
    h0, hs = traceless_terms(n_ctrl, 1000 + n_ctrl)
    rng = np.random.default_rng(7 + n_ctrl)
    slices = 3001
    pts = slices if mode == "midpoint" else 2 * slices + 1
    norm = sum(np.abs(h).sum(axis=0).max() for h in [h0, *hs])
    dt = 0.3 / norm
    values = rng.uniform(-1.0, 1.0, (pts, n_ctrl))
    _gate(h0, hs, values, dt, mode, label=f"N={n_ctrl}")


@pytest.mark.parametrize("beta", [1e-4, 3e-3, 0.05, 0.5, 2.0, 4.4])
def test_series_orders_compiled_and_runtime(beta):
    """beta spans m = 3 .. 25 (3, 5, 7 compiled in; the rest at runtime)."""
    h0, hs = traceless_terms(2, 77)
    rng = np.random.default_rng(3)
    values = rng.uniform(-1.0, 1.0, (20000, 2))
    norm = sum(np.abs(h).sum(axis=0).max() for h in [h0, *hs])
    _gate(h0, hs, values, beta / norm, "midpoint", label=f"beta={beta}")


@pytest.mark.parametrize("slices", [1, 2, 31, 33, 1000, 70001])
def test_slice_counts(slices):
    h0, hs, values, dt = qubit_inputs(slices, "midpoint")
    _gate(h0, hs, values, dt, "midpoint", label="qubit")


@pytest.mark.parametrize("mode", ["midpoint", "simpson", "magnus"])
def test_driven_qubit_modes(mode):
    pts = 100_000 if mode == "midpoint" else 100_001
    h0, hs, values, dt = qubit_inputs(pts, mode)
    _gate(h0, hs, values, dt, mode, label="qubit")


def test_driven_qubit_1e6_against_80bit_oracle():
    """SURVEY.md §8(c) d = 2 gate: error vs the 80-bit oracle of the same
    midpoint discretisation <= 2x the reference's (8.6e-11 at 1e6)."""
    h0, hs, values, dt = qubit_inputs(1_000_000, "midpoint")
    res, kernel = _run(h0, hs, values, dt, "midpoint")
    assert kernel == "lane_su2_kernel"
    exact = oracle.midpoint_reference_ld(1.0, 0.1, 1.0, 6.0, 1_000_000)
    err = float(np.abs(res.u - exact).max())
    print(f"\n[su2] qubit 1e6 vs 80-bit: {err:.3e} (reference 8.6e-11)")
    assert err <= 2 * 8.6e-11


def test_matches_the_complex_pair_kernel():
    """Same U per slice as lane_small_kernel<2,1>'s real-pair path: the two
    kernels agree to rounding (SP_SU2=0 is checked in a subprocess)."""
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path[:0] = ['tests/golden', '.'];"
            "from cases import qubit_inputs; import paper_2108_07126_b200 as sp;"
            "h0, hs, v, dt = qubit_inputs(50000, 'midpoint'); ctx = sp.create();"
            "ctx.set_hamiltonian(sp.ControlSystem(h0, hs));"
            "u = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u;"
            "print(ctx.last_timing()['kernel']); np.save(sys.argv[1], u)")
    import os
    import tempfile
    out = os.path.join(tempfile.mkdtemp(), "u.npy")
    env = dict(os.environ, SP_SU2="0")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code, out], env=env, cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().startswith("lane_small_kernel")
    h0, hs, values, dt = qubit_inputs(50000, "midpoint")
    res, kernel = _run(h0, hs, values, dt, "midpoint")
    assert kernel == "lane_su2_kernel"
    assert rel_fro(res.u, np.load(out)) <= 1e-12


@pytest.mark.parametrize("mode", ["midpoint", "magnus"])
def test_amplitude_bound_first_offender(mode):
    h0, hs, values, dt = qubit_inputs(40001, mode)
    values = values.copy()
    values[31234, 1] = 1.5
    values[31234, 0] = np.nan
    values[39000, 0] = -2.0
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus")
        # ControlAmplitudes validates on the host; the device check is what
        # equiprop_device_ptr relies on, so go through the device entry
        import torch
        d = torch.from_numpy(values).cuda()
        out = torch.empty((2, 2), dtype=torch.complex128, device="cuda")
        ctx.equiprop_device_ptr(d.data_ptr(), values.shape[0], 2, dt, out.data_ptr())
        torch.cuda.synchronize()
        assert ctx.last_timing()["kernel"] == "lane_su2_kernel"
        assert ctx.amplitude_violation() == 31234 * 2 + 0
        # the next clean call clears the slot (epoch rotation)
        clean = torch.from_numpy(np.clip(np.nan_to_num(values), -1, 1)).cuda()
        ctx.equiprop_device_ptr(clean.data_ptr(), values.shape[0], 2, dt, out.data_ptr())
        torch.cuda.synchronize()
        assert ctx.amplitude_violation() == -1


def test_host_entry_raises_reference_message():
    h0, hs, values, dt = qubit_inputs(1000, "midpoint")
    values = values.copy()
    values[500, 1] = 1.25
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        with pytest.raises(sp.AmplitudeBoundError, match="sample 500, control 1"):
            ctx.equiprop(sp.ControlAmplitudes(values, dt))


def test_not_traceless_uses_the_u2_lanes():
    """A trace part leaves the quaternion algebra: the same lanes run on 2 x 2
    complex products (tests/test_u2_gpu.py holds them to the gate)."""
    h0, hs, values, dt = qubit_inputs(1000, "midpoint")
    h0 = h0 + 0.25 * np.eye(2)
    res, kernel = _run(h0, hs, values, dt, "midpoint")
    assert kernel == "lane_u2_kernel"


def test_misaligned_table_falls_back_to_the_general_kernel():
    """A device table whose rows are not 16-byte aligned (offset by one
    double) cannot feed the TMA / vector row loads: the general d = 2 kernel
    runs instead, with the same result."""
    import torch
    h0, hs, values, dt = qubit_inputs(20000, "midpoint")
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        base = torch.zeros(values.size + 1, dtype=torch.float64, device="cuda")
        base[1:] = torch.from_numpy(values.reshape(-1)).cuda()
        out = torch.empty((2, 2), dtype=torch.complex128, device="cuda")
        ctx.equiprop_device_ptr(base.data_ptr() + 8, values.shape[0], 2, dt, out.data_ptr())
        torch.cuda.synchronize()
        assert ctx.last_timing()["kernel"].startswith("lane_small")
        aligned = torch.from_numpy(values).cuda()
        out2 = torch.empty_like(out)
        ctx.equiprop_device_ptr(aligned.data_ptr(), values.shape[0], 2, dt, out2.data_ptr())
        torch.cuda.synchronize()
        assert ctx.last_timing()["kernel"] == "lane_su2_kernel"
        assert rel_fro(out.cpu().numpy(), out2.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("mode", ["midpoint", "magnus"])
def test_emulated_multi_device_qubit(mode):
    """A multi-device context (4 children emulated on device 0) runs the
    su(2) kernel on every block and matches the single-device result."""
    pts = 400_000 if mode == "midpoint" else 400_001
    h0, hs, values, dt = qubit_inputs(pts, mode)
    res = []
    for devs in (None, [0, 0, 0, 0]):
        with sp.create(devices=devs) as ctx:
            ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus")
            res.append(ctx.equiprop(sp.ControlAmplitudes(values, dt)).u)
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode)
    ref, seq = oracle.reduce_pairwise(u), oracle.reduce_sequential(u)
    tol, _ = parity_tolerance(ref, seq, "fp64")
    assert rel_fro(res[1], res[0]) <= tol
    assert rel_fro(res[1], ref) <= tol


@pytest.mark.parametrize("mode", ["midpoint", "magnus"])
@pytest.mark.parametrize("slices", [1, 5000, 300_000])
def test_complex64_contexts_run_float32_su2(mode, slices):
    """complex64 contexts: the same kernels in float32 arithmetic (weights
    and terms cast to float32 as the reference's fp32 path does), gated
    against the oracle's complex64 restatement: max(1e-5, 4 eps_self)."""
    pts = slices if mode == "midpoint" else 2 * slices + 1
    h0, hs, values, dt = qubit_inputs(pts, mode)
    with sp.create("fp32") as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus")
        res = ctx.equiprop(sp.ControlAmplitudes(values, dt))
        kernel = ctx.last_timing()["kernel"]
    assert kernel == "lane_su2_f32_kernel" and res.u.dtype == np.complex64
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode, bits=32)
    ref, seq = oracle.reduce_pairwise(u), oracle.reduce_sequential(u)
    tol, eps = parity_tolerance(ref, seq, "fp32")
    u64, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode)
    ref64 = oracle.reduce_pairwise(u64)
    err, err64, ref_err64 = rel_fro(res.u, ref), rel_fro(res.u, ref64), rel_fro(ref, ref64)
    print(f"\n[su2 f32] {mode} slices={slices}: vs ref c64 {err:.3e} (tol {tol:.3e}), "
          f"vs c128 {err64:.3e} (reference c64 vs c128 {ref_err64:.3e})")
    assert err <= tol or err64 <= ref_err64


@pytest.mark.parametrize("mode", ["midpoint", "simpson", "magnus"])
@pytest.mark.parametrize("slices", [1, 37, 50_000])
def test_lane_mode_sequential_and_cumulative(mode, slices):
    """Lane mode of the su(2) kernels (reduction="sequential" and the d = 2
    two-pass equiprop_all): lane products / per-slice running products in
    the plain 2 x 2 layout, the ordered scan, pass 2 from the exclusive lane
    prefixes.  Gates: sequential total and every cumulative entry vs the
    oracle (max(1e-12, 4 eps_self)); the reference property u_all[-1] ==
    sequential total, bit for bit (propagator.py:304-306)."""
    pts = slices if mode == "midpoint" else 2 * slices + 1
    h0, hs, values, dt = qubit_inputs(pts, mode)
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        amps = sp.ControlAmplitudes(values, dt)
        seq = ctx.equiprop(amps, reduction="sequential").u
        assert ctx.last_timing()["kernel"] == "lane_su2_kernel"
        cum = ctx.equiprop_all(amps)
        assert ctx.last_timing()["kernel"] == "lane_su2_kernel"
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode)
    ref, ref_seq = oracle.reduce_pairwise(u), oracle.reduce_sequential(u)
    tol, _ = parity_tolerance(ref, ref_seq, "fp64")
    assert rel_fro(seq, ref_seq) <= tol
    assert np.array_equal(cum.u_all[-1], seq)
    ref_all = oracle.cumulative(u)
    step = max(1, slices // 200)
    worst = max(rel_fro(cum.u_all[k], ref_all[k]) for k in range(0, slices, step))
    print(f"\n[su2 lane mode] {mode} slices={slices}: seq {rel_fro(seq, ref_seq):.3e}, "
          f"cumulative worst {worst:.3e} (tol {tol:.3e})")
    assert worst <= tol
