"""Public-API behaviour that needs the device (reference tests/test_propagator.py
TestEquiprop / TestLifecycle / TestMagnusMode / TestEquipropAll and
bindings/tests/test_binding.py, run against the B200 path)."""

import numpy as np
import pytest

import paper_2108_07126_b200 as sp
from paper_2108_07126_b200 import pysliceprop
from helpers import expm_eigh, haar_unitary, random_hermitian

pytestmark = pytest.mark.gpu

SZ = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=complex)
SX = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)
SY = np.array([[0.0, -1.0j], [1.0j, 0.0]], dtype=complex)


def drift_qubit():
    return sp.ControlSystem(SZ / 2.0)


def driven_qubit():
    return sp.ControlSystem(SZ / 2.0, [SX / 2.0, SY / 2.0])


def driven_amps(pts, dt=0.02, wrf=1.0):
    t = np.arange(pts) * dt
    return sp.ControlAmplitudes(np.column_stack([np.cos(wrf * t), np.sin(wrf * t)]), dt)


def sequential_product(mats):
    acc = np.eye(mats[0].shape[0], dtype=complex)
    for m in mats:
        acc = m @ acc
    return acc


def dense_reference(system, amps, quadrature="midpoint"):
    if quadrature == "midpoint":
        slices = [amps.dt * (system.drift + sum(c * h for c, h in zip(row, system.controls)))
                  for row in amps.values]
    else:
        v = amps.values
        avg = (v[0:-1:2] + 4.0 * v[1::2] + v[2::2]) / 6.0
        slices = [2.0 * amps.dt * (system.drift + sum(c * h for c, h in zip(row, system.controls)))
                  for row in avg]
    return sequential_product([expm_eigh(g) for g in slices])


@pytest.mark.parametrize("d", [2, 4, 16, 32, 64, 128])
def test_amplitude_violation_raised_from_device(d, rng):
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(random_hermitian(rng, d, 1.0),
                                         [random_hermitian(rng, d, 1.0)] * 2))
    values = np.zeros((40, 2))
    values[25, 1] = 1.5
    values[31, 0] = -2.0
    with pytest.raises(sp.AmplitudeBoundError, match=r"1\.5 at sample 25, control 1"):
        ctx.equiprop(sp.ControlAmplitudes(values, 0.01))
    values[25, 1] = np.nan
    with pytest.raises(sp.AmplitudeBoundError, match="sample 25, control 1"):
        ctx.equiprop_all(sp.ControlAmplitudes(values, 0.01))
    # the context stays usable
    values[25, 1] = 0.0
    values[31, 0] = 0.0
    u = ctx.equiprop(sp.ControlAmplitudes(values, 0.01)).u
    assert np.allclose(u.conj().T @ u, np.eye(d), atol=1e-12)


def test_three_point_violation_found_in_shared_endpoints():
    ctx = sp.create()
    ctx.set_hamiltonian(driven_qubit(), magnus=True)
    values = driven_amps(21).values.copy()
    values[20, 1] = 1.0000001
    with pytest.raises(sp.AmplitudeBoundError, match="sample 20, control 1"):
        ctx.equiprop(sp.ControlAmplitudes(values, 0.1))


def test_constant_drift_closed_form():
    ctx = sp.create()
    ctx.set_hamiltonian(drift_qubit())
    result = ctx.equiprop(sp.ControlAmplitudes(np.zeros((10, 0)), 0.1))
    assert np.abs(result.u - np.diag([np.exp(-0.5j), np.exp(0.5j)])).max() <= 1e-12
    assert result.slice_count == 10


def test_zero_hamiltonian_is_exact_identity():
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(np.zeros((2, 2))))
    assert np.array_equal(ctx.equiprop(sp.ControlAmplitudes(np.zeros((6, 0)), 0.3)).u,
                          np.eye(2))
    ctx.set_hamiltonian(sp.ControlSystem(np.zeros((40, 40))))
    assert np.array_equal(ctx.equiprop(sp.ControlAmplitudes(np.zeros((6, 0)), 0.3)).u,
                          np.eye(40))


def test_driven_qubit_and_simpson_against_dense_reference():
    system = driven_qubit()
    amps = driven_amps(25)
    ctx = sp.create()
    ctx.set_hamiltonian(system)
    assert np.abs(ctx.equiprop(amps).u - dense_reference(system, amps)).max() <= 1e-12
    ctx.set_hamiltonian(system, quadrature="simpson")
    res = ctx.equiprop(amps)
    assert np.abs(res.u - dense_reference(system, amps, "simpson")).max() <= 1e-12
    assert res.slice_count == 12


def test_composition_of_halves():
    system = driven_qubit()
    full = driven_amps(40)
    ctx = sp.create()
    ctx.set_hamiltonian(system)
    first = sp.ControlAmplitudes(full.values[:20], full.dt)
    second = sp.ControlAmplitudes(full.values[20:], full.dt)
    u_halves = ctx.equiprop(second).u @ ctx.equiprop(first).u
    assert np.abs(ctx.equiprop(full).u - u_halves).max() <= 1e-12


def test_reload_replaces_system_and_dimension(rng):
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(SZ * np.pi / 2.0))
    amps = sp.ControlAmplitudes(np.zeros((1, 0)), 1.0)
    assert np.allclose(ctx.equiprop(amps).u, np.diag([-1j, 1j]), atol=1e-13)
    ctx.set_hamiltonian(sp.ControlSystem(SX * np.pi / 2.0))
    assert np.allclose(ctx.equiprop(amps).u, -1j * SX, atol=1e-13)
    ctx.set_hamiltonian(sp.ControlSystem(random_hermitian(rng, 7, norm=1.0)))
    assert ctx.equiprop(sp.ControlAmplitudes(np.zeros((3, 0)), 0.1)).u.shape == (7, 7)


def test_contexts_are_independent():
    a = sp.create(precision="fp64")
    b = sp.create(precision="fp32")
    a.set_hamiltonian(drift_qubit())
    b.set_hamiltonian(drift_qubit())
    amps = sp.ControlAmplitudes(np.zeros((5, 0)), 0.1)
    assert a.equiprop(amps).u.dtype == np.complex128
    assert b.equiprop(amps).u.dtype == np.complex64


def test_magnus_agrees_with_simpson_on_commuting_problem():
    system = sp.ControlSystem(SZ / 2.0, [SZ / 4.0])
    amps = sp.ControlAmplitudes(np.linspace(-1.0, 1.0, 11)[:, None], 0.05)
    m = sp.create()
    m.set_hamiltonian(system, magnus=True)
    s = sp.create()
    s.set_hamiltonian(system, quadrature="simpson")
    assert np.abs(m.equiprop(amps).u - s.equiprop(amps).u).max() <= 1e-13


def test_magnus_plan_uses_commutator_bound():
    system = driven_qubit()
    ctx = sp.create()
    ctx.set_hamiltonian(system, magnus=True)
    amps = driven_amps(9)
    expected = sp.magnus_spectral_bound(sp.build_effective_system(system), amps)
    assert ctx.equiprop(amps).plan["beta"] == pytest.approx(expected)


def test_equiprop_all_contract():
    ctx = sp.create()
    ctx.set_hamiltonian(driven_qubit())
    amps = driven_amps(12)
    cum = ctx.equiprop_all(amps)
    assert cum.u_all.shape == (12, 2, 2) and cum.slice_count == 12
    single = ctx.equiprop(sp.ControlAmplitudes(amps.values[:1], amps.dt)).u
    assert np.abs(cum.u_all[0] - single).max() <= 1e-15
    assert np.array_equal(cum.final, ctx.equiprop(amps, reduction="sequential").u)
    for k in (2, 5, 8):
        prefix = sp.ControlAmplitudes(amps.values[:k + 1], amps.dt)
        assert np.abs(cum.u_all[k] - ctx.equiprop(prefix, reduction="sequential").u).max() \
            <= 1e-14
    for u in cum.u_all:
        assert sp.one_norm(u.conj().T @ u - np.eye(2)) <= 1e-11
    ctx.set_hamiltonian(driven_qubit(), magnus=True)
    assert ctx.equiprop_all(driven_amps(11)).u_all.shape == (5, 2, 2)


def test_fp32_pipeline():
    ctx = sp.create(precision="fp32")
    ctx.set_hamiltonian(driven_qubit())
    u = ctx.equiprop(driven_amps(21)).u
    assert u.dtype == np.complex64
    assert sp.one_norm(u.conj().T @ u - np.eye(2)) <= 1e-4


@pytest.mark.parametrize("n", [1, 2, 3, 7, 8, 33, 64, 257, 1000])
def test_reduction_all_counts(rng, n):
    """Ordered products at awkward counts (odd carries, single lanes)."""
    d = 4
    h = random_hermitian(rng, d, norm=1.0)
    c = random_hermitian(rng, d, norm=1.0)
    values = rng.uniform(-1, 1, (n, 1))
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h, [c]))
    amps = sp.ControlAmplitudes(values, 0.1)
    ref = sequential_product([expm_eigh(0.1 * (h + v[0] * c)) for v in values])
    for red in ("pairwise", "sequential"):
        assert np.abs(ctx.equiprop(amps, reduction=red).u - ref).max() <= 1e-13


def test_binding_session_and_errors():
    problem = dict(drift=0.5 * np.kron(SZ, np.eye(2)), controls=[0.5 * np.kron(SX, np.eye(2))],
                   c=0.7 * np.cos(np.arange(21) * 0.05)[:, None], dt=0.05)
    u = pysliceprop.equiprop(problem["drift"], problem["controls"], problem["c"], problem["dt"],
                             magnus=True)
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(problem["drift"], problem["controls"]), magnus=True)
    assert np.array_equal(u, ctx.equiprop(sp.ControlAmplitudes(problem["c"], 0.05)).u)
    with pysliceprop.Session() as s:
        s.set_hamiltonian(SZ / 2, [SX / 2])
        with pytest.raises(pysliceprop.BindingError) as ei:
            s.equiprop(np.full((5, 1), 3.0), 0.1)
        assert ei.value.code == "amplitude-bound"
        cum = s.equiprop(np.zeros((4, 1)), 0.1, cumulative=True)
        assert cum.shape == (4, 2, 2)


@pytest.mark.parametrize("d", [2, 8, 32])
def test_equiprop_all_device_matches_host(d, rng):
    """sp_equiprop_all_device (device-resident table and output, caller's
    stream) returns exactly the host entry's cumulative stack."""
    import torch
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(random_hermitian(rng, d, 1.0),
                                         [random_hermitian(rng, d, 1.0)] * 2))
    values = rng.uniform(-1.0, 1.0, (300, 2))
    amps = sp.ControlAmplitudes(values, 0.05)
    host = ctx.equiprop_all(amps).u_all
    dev = torch.device("cuda", 0)
    d_amps = torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    out = torch.empty((300, d, d), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    info = ctx.equiprop_all_device_ptr(d_amps.data_ptr(), 300, 2, 0.05, out.data_ptr(),
                                       stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    assert info["slice_count"] == 300
    assert np.array_equal(out.cpu().numpy(), host)
    ctx.close()


@pytest.mark.parametrize("n", [0, 1, 2, 5, 33, 64])
@pytest.mark.parametrize("dtype", [np.complex128, np.complex64])
def test_reduce_pairwise_matches_reference_order(n, dtype, rng):
    """Module-level reduce_pairwise (propagator.py:68-102) on the device
    against the reference's level-order fold restated by the oracle; the
    empty batch is the identity."""
    import oracle
    d = 3
    u = np.stack([haar_unitary(rng, d) for _ in range(n)]).astype(dtype) if n else \
        np.zeros((0, d, d), dtype=dtype)
    got = sp.reduce_pairwise(u)
    assert got.dtype == dtype and got.shape == (d, d)
    if n == 0:
        assert np.array_equal(got, np.eye(d, dtype=dtype))
        return
    ref = oracle.reduce_pairwise(u.astype(np.complex128))
    tol = 1e-13 if dtype == np.complex128 else 1e-5
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= tol


@pytest.mark.parametrize("d", [2, 4])
def test_violation_slots_across_fused_calls_and_graph_replays(d, rng):
    """Single-launch calls (small families, pairwise) record violations in
    epoch-rotated slots instead of a memset in front of the launch: every
    call, fused or not, replayed in a CUDA graph or not, reports exactly its
    own first offender."""
    import torch
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(random_hermitian(rng, d, 1.0),
                                         [random_hermitian(rng, d, 1.0)] * 2))
    dev = torch.device("cuda", 0)
    good = rng.uniform(-1.0, 1.0, (500, 2))
    bad = good.copy()
    bad[321, 1] = 1.25
    worse = good.copy()
    worse[17, 0] = np.nan
    # host entry points: fused (pairwise) and multi-launch (sequential,
    # cumulative) interleaved with and without violations
    seq = [(good, "pairwise", None), (bad, "pairwise", 321 * 2 + 1), (good, "pairwise", None),
           (bad, "sequential", 321 * 2 + 1), (good, "pairwise", None), (worse, "all", 34),
           (good, "pairwise", None), (good, "sequential", None), (worse, "pairwise", 34),
           (bad, "pairwise", 321 * 2 + 1), (good, "all", None), (good, "pairwise", None)]
    for values, kind, expect in seq:
        amps = sp.ControlAmplitudes(values, 0.02)
        call = (lambda: ctx.equiprop_all(amps)) if kind == "all" else \
            (lambda: ctx.equiprop(amps, reduction=kind))
        if expect is None:
            call()
        else:
            with pytest.raises(sp.AmplitudeBoundError,
                               match=f"sample {expect // 2}, control {expect % 2}"):
                call()
    # device entry point captured once and replayed with new table contents
    d_amps = torch.from_numpy(np.ascontiguousarray(good)).to(dev)
    out = torch.empty((d, d), dtype=torch.complex128, device=dev)
    plan = ctx.plan_for(0.02)
    s = torch.cuda.Stream(dev)
    ctx.set_profiling(False)
    ctx.equiprop_device_ptr(d_amps.data_ptr(), 500, 2, 0.02, out.data_ptr(),
                            stream=s.cuda_stream, plan=plan)
    assert ctx.amplitude_violation() == -1
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.equiprop_device_ptr(d_amps.data_ptr(), 500, 2, 0.02, out.data_ptr(),
                                stream=s.cuda_stream, plan=plan)
    for values, expect in ((good, -1), (bad, 321 * 2 + 1), (bad, 321 * 2 + 1), (good, -1),
                           (worse, 34), (good, -1), (good, -1), (bad, 643)):
        d_amps.copy_(torch.from_numpy(np.ascontiguousarray(values)))
        g.replay()
        torch.cuda.synchronize(dev)
        assert ctx.amplitude_violation() == expect
    ctx.close()


def test_more_than_2_31_slices_device_resident():
    """64-bit slice indexing: 3 * 2^30 slices (a 51 GB table in HBM; row
    index x controls > 2^32), the drive switching at row 2^31, against the
    closed form exp(-i T2 H2) exp(-i T1 H1): rows past 2^31 read wrongly
    (an int32 wrap) would change the result at O(1)."""
    import torch
    n1, n = 1 << 31, 3 << 30
    dt = 3e-10
    c1, c2 = (0.3, -0.4), (-0.8, 0.5)
    ctx = sp.create()
    sysm = driven_qubit()
    ctx.set_hamiltonian(sysm)
    dev = torch.device("cuda", 0)
    d_amps = torch.empty((n, 2), dtype=torch.float64, device=dev)
    d_amps[:n1, 0], d_amps[:n1, 1] = c1
    d_amps[n1:, 0], d_amps[n1:, 1] = c2
    out = torch.empty((2, 2), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    info = ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                   stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    assert info["slice_count"] == n
    assert ctx.amplitude_violation() == -1
    h1 = sysm.drift + c1[0] * sysm.controls[0] + c1[1] * sysm.controls[1]
    h2 = sysm.drift + c2[0] * sysm.controls[0] + c2[1] * sysm.controls[1]
    ref = expm_eigh((n - n1) * dt * h2) @ expm_eigh(n1 * dt * h1)
    got = out.cpu().numpy()
    # identical slices repeat the same rounding: the error grows ~ n eps
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-5
    # a violation past the 2^32 index boundary is reported at its row
    d_amps[n - 3, 1] = 1.5
    ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                            stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    assert ctx.amplitude_violation() == (n - 3) * 2 + 1
    del d_amps
    torch.cuda.empty_cache()
    ctx.close()


def test_complex64_d2_register_lanes_match_the_two_thread_lanes():
    """lane_f32_reg2_kernel (one thread per d = 2 lane, registers only) runs
    the same per-column float32 operation sequence as the two-thread
    lane_f32_kernel<2>: bitwise-identical lane products (SP_F32_REG2=0 in a
    subprocess selects the two-thread form)."""
    import os
    import subprocess
    import sys
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import numpy as np, sys; sys.path[:0] = ['tests/golden', '.'];"
            "from cases import random_inputs; import paper_2108_07126_b200 as sp;"
            "h0, hs, v, dt = random_inputs(2, 2, 40000, 9); ctx = sp.create('fp32');"
            "ctx.set_hamiltonian(sp.ControlSystem(h0, hs));"
            "u = ctx.equiprop(sp.ControlAmplitudes(v, dt), reduction='sequential').u;"
            "print(ctx.last_timing()['kernel']); np.save(sys.argv[1], u)")
    outs = []
    for flag in ("1", "0"):
        out = os.path.join(tempfile.mkdtemp(), "u.npy")
        r = subprocess.run([sys.executable, "-c", code, out], cwd=root, capture_output=True,
                           text=True, timeout=300, env=dict(os.environ, SP_F32_REG2=flag))
        assert r.returncode == 0, r.stderr
        outs.append(np.load(out))
    assert np.array_equal(outs[0], outs[1])
