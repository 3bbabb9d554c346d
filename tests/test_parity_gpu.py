"""GPU parity: the sm_100a path (through the public API, i.e. the C ABI)
against the reference outputs committed in tests/golden/ and against the CPU
oracle on the same seeded inputs.

Tolerance: rel-Frobenius(U_gpu, U_ref) <= max(floor,
4 eps_self), floor = 1e-12 (complex128) / 1e-5 (complex64), eps_self = the
reference's own pairwise-vs-sequential difference on the same input.
"""

import json
import os

import numpy as np
import pytest

from cases import CASES, CONVERGE_PTS, build_inputs, input_digest
from helpers import parity_tolerance, rel_fro

import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _run(case, reduction="pairwise"):
    h0, hs, values, dt = build_inputs(case)
    mode = case["mode"]
    ctx = sp.create(precision=case["precision"], m_max=case.get("m_max"))
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    amps = sp.ControlAmplitudes(values, dt)
    res = ctx.equiprop(amps, reduction=reduction)
    return ctx, amps, res, (h0, hs, values, dt)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_equiprop_matches_reference(case, golden):
    key = case["name"]
    ctx, amps, res, inputs = _run(case)
    assert bytes(golden[f"{key}__digest"]) == input_digest(*inputs)
    u_ref = golden[f"{key}__u"]
    tol, eps_self = parity_tolerance(u_ref, golden[f"{key}__u_seq"], case["precision"])
    err = rel_fro(res.u, u_ref)
    assert res.u.dtype == u_ref.dtype
    assert res.slice_count == int(golden[f"{key}__slice_count"])
    if f"{key}__m_max" in golden.files:
        assert res.plan["m_max"] == int(golden[f"{key}__m_max"])
        assert res.plan["beta"] == pytest.approx(float(golden[f"{key}__beta"]), rel=1e-15)
    assert err <= tol, f"{key}: err {err:.3e} > tol {tol:.3e} (eps_self {eps_self:.3e})"
    # sequential reduction obeys the same gate
    u_seq = ctx.equiprop(amps, reduction="sequential").u
    assert rel_fro(u_seq, u_ref) <= tol
    if case.get("cumulative"):
        cum = ctx.equiprop_all(amps)
        ref_all = golden[f"{key}__u_all"]
        assert cum.u_all.shape == ref_all.shape
        for k in range(ref_all.shape[0]):
            assert rel_fro(cum.u_all[k], ref_all[k]) <= tol, k
        # reference property propagator.py:304-306: last entry == sequential
        assert np.array_equal(cum.final, u_seq)
    ctx.close()


@pytest.mark.parametrize("case", [c for c in CASES if c["kind"] == "random"][:12],
                         ids=lambda c: c["name"])
def test_deterministic(case):
    ctx, amps, res, _ = _run(case)
    again = ctx.equiprop(amps).u
    assert np.array_equal(res.u, again)
    ctx.close()


def test_convergence_orders_reproduced():
    """C2: the dt sweep of the driven qubit on the GPU reproduces the
    reference's errors where truncation dominates and its fitted orders
    (bands of reference test_acceptance.py:133-145)."""
    with open(os.path.join(HERE, "golden", "converge.json")) as fh:
        gold = json.load(fh)
    problem = sp.DrivenQubit(1.0, 0.1, 1.0, 6.0)
    bands = {"midpoint": (1.9, 2.2), "simpson": (1.9, 2.2), "magnus": (3.7, 4.3)}
    for label, magnus, quad in [("midpoint", False, "midpoint"),
                                ("simpson", False, "simpson"),
                                ("magnus", True, None)]:
        rows = sp.convergence_sweep(problem, CONVERGE_PTS, magnus=magnus, quadrature=quad)
        pts = [p for p, _ in rows]
        errs = np.array([e for _, e in rows])
        ref = np.array(gold[label]["errors"])
        assert pts == gold[label]["pts"]
        # truncation-dominated points agree to 1e-4 relative (+ roundoff floor)
        assert np.all(np.abs(errs - ref) <= 1e-4 * ref + 5e-11), (label, errs, ref)
        order, _ = sp.fit_convergence_order(pts, errs)
        lo, hi = bands[label]
        assert lo <= order <= hi, (label, order)
        assert abs(order - gold[label]["order"]) < 0.05, (label, order, gold[label]["order"])


TC_CASES = [c for c in CASES if c["kind"] != "zero" and c.get("d", 2) >= 5]


@pytest.mark.parametrize("algo", ["clenshaw", "ps", "ps3m"])
@pytest.mark.parametrize("case", TC_CASES, ids=[c["name"] for c in TC_CASES])
def test_both_series_schemes_match_reference(case, algo, golden):
    """The tensor-core families evaluate the same plan polynomial either by
    the reference's Clenshaw recurrence or by Paterson-Stockmeyer in the
    Chebyshev basis; both pass the same gate."""
    key = case["name"]
    h0, hs, values, dt = build_inputs(case)
    mode = case["mode"]
    ctx = sp.create(precision=case["precision"], m_max=case.get("m_max"))
    ctx.set_algorithm(algo)
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    amps = sp.ControlAmplitudes(values, dt)
    u = ctx.equiprop(amps).u
    # complex64 contexts of the plain families (d <= 8) compute in complex64
    # arithmetic with the reference's Clenshaw recurrence whatever the scheme
    f32 = case["precision"] == "fp32" and case.get("d", 2) <= 8
    assert ctx.last_algorithm()["algorithm"] == ("clenshaw_fp32" if f32 else algo)
    tol, _ = parity_tolerance(golden[f"{key}__u"], golden[f"{key}__u_seq"], case["precision"])
    assert rel_fro(u, golden[f"{key}__u"]) <= tol
    if case.get("cumulative"):
        cum = ctx.equiprop_all(amps)
        for k in range(cum.u_all.shape[0]):
            assert rel_fro(cum.u_all[k], golden[f"{key}__u_all"][k]) <= tol
        assert np.array_equal(cum.final, ctx.equiprop(amps, reduction="sequential").u)
    ctx.close()


@pytest.mark.parametrize("d,n_ctrl,pts,mode", [(200, 2, 6, "midpoint"), (300, 3, 5, "simpson"),
                                               (512, 2, 4, "midpoint"), (384, 2, 5, "magnus")])
@pytest.mark.parametrize("algo", ["auto", "clenshaw", "ps"])
def test_large_dims_against_oracle(d, n_ctrl, pts, mode, algo):
    """d > 128 (families D256/D512) against the CPU oracle (bit-exact
    restatement of the reference) on the same inputs."""
    import oracle
    from cases import random_inputs
    h0, hs, values, dt = random_inputs(d, n_ctrl, pts, 4242 + d)
    ref, n, _ = oracle.equiprop(h0, hs, values, dt, mode=mode)
    ref_seq, _, _ = oracle.equiprop(h0, hs, values, dt, mode=mode, reduction="sequential")
    tol, _ = parity_tolerance(ref, ref_seq, "fp64")
    ctx = sp.create()
    ctx.set_algorithm(algo)
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    res = ctx.equiprop(sp.ControlAmplitudes(values, dt))
    assert res.slice_count == n
    assert rel_fro(res.u, ref) <= tol
    ctx.close()


@pytest.mark.parametrize("pts", [1, 37, 5000, 200_000])
@pytest.mark.parametrize("hermitian_exact", [True, False])
def test_d2_paths_against_oracle(pts, hermitian_exact):
    """d = 2 runs the reference's Clenshaw recurrence on Cayley-Hamilton
    coefficient pairs: with real coefficients when every term is bitwise
    Hermitian, complex ones otherwise (an asymmetry far inside the
    reference's 1e-12 ingest tolerance).  Both against the oracle, from one
    slice up to several slices per lane and the multi-CTA fused tail."""
    import oracle
    from cases import random_inputs
    h0, hs, values, dt = random_inputs(2, 2, pts, 99 + pts)
    if not hermitian_exact:
        hs[0] = hs[0].copy()
        hs[0][0, 1] += 1e-15
    ref, _, _ = oracle.equiprop(h0, hs, values, dt, mode="midpoint")
    ref_seq, _, _ = oracle.equiprop(h0, hs, values, dt, mode="midpoint", reduction="sequential")
    tol, _ = parity_tolerance(ref, ref_seq, "fp64")
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    amps = sp.ControlAmplitudes(values, dt)
    assert rel_fro(ctx.equiprop(amps).u, ref) <= tol
    assert rel_fro(ctx.equiprop(amps, reduction="sequential").u, ref) <= tol
    ctx.close()


@pytest.mark.parametrize("d", [1, 2, 3, 6, 8, 12, 24, 40, 96])
@pytest.mark.parametrize("mode", ["midpoint", "simpson", "magnus"])
def test_cumulative_every_family_against_oracle(d, mode):
    """equiprop_all for every kernel family (plain-layout d <= 8, DMMA
    prefix application above) against the oracle's cumulative stack, and the
    reference property u_all[-1] == sequential total, bit for bit
    (propagator.py:304-306, 310-316)."""
    import oracle
    from cases import random_inputs
    h0, hs, values, dt = random_inputs(d, 2, 41, 7000 + d)
    ref_all, _, _ = oracle.equiprop_all(h0, hs, values, dt, mode=mode)
    ref, _, _ = oracle.equiprop(h0, hs, values, dt, mode=mode)
    ref_seq, _, _ = oracle.equiprop(h0, hs, values, dt, mode=mode, reduction="sequential")
    tol, _ = parity_tolerance(ref, ref_seq, "fp64")
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    amps = sp.ControlAmplitudes(values, dt)
    cum = ctx.equiprop_all(amps)
    assert cum.u_all.shape == ref_all.shape
    for k in range(ref_all.shape[0]):
        assert rel_fro(cum.u_all[k], ref_all[k]) <= tol, k
    assert np.array_equal(cum.final, ctx.equiprop(amps, reduction="sequential").u)
    ctx.close()


@pytest.mark.parametrize("pts,algo", [(200, "auto"), (200, "ps"), (2001, "auto")])
def test_spin_chain_against_oracle(pts, algo):
    """BASELINE configs[2]: the 5-spin coupled chain (d = 32, 2 controls)
    against the oracle, plus unitarity of the propagator."""
    import oracle
    chain = sp.SpinChain()
    system = chain.system()
    amps = chain.amplitudes(pts)
    h0, hs = system.drift, list(system.controls)
    ref, _, _ = oracle.equiprop(h0, hs, amps.values, amps.dt, mode="midpoint")
    ref_seq, _, _ = oracle.equiprop(h0, hs, amps.values, amps.dt, mode="midpoint",
                                    reduction="sequential")
    tol, _ = parity_tolerance(ref, ref_seq, "fp64")
    ctx = sp.create()
    ctx.set_algorithm(algo)
    ctx.set_hamiltonian(system)
    u = ctx.equiprop(amps).u
    assert rel_fro(u, ref) <= tol
    # unitarity no worse than the reference's own (rounding accumulates with n)
    dev = lambda m: np.linalg.norm(m.conj().T @ m - np.eye(32))
    assert dev(u) <= max(1e-12, 4.0 * dev(ref))
    ctx.close()


@pytest.mark.parametrize("m", list(range(3, 26, 2)))
@pytest.mark.parametrize("d", [3, 4])
def test_small_family_every_series_order_against_oracle(d, m):
    """d = 3, 4 compile the series order in for every order of the plan grid
    (and use the plan's alternating real / imaginary coefficients): each
    order against the oracle with the same pinned m, pairwise and
    cumulative."""
    import oracle
    from cases import random_inputs
    h0, hs, values, dt = random_inputs(d, 2, 300, 500 + 10 * d + m)
    ref, _, plan = oracle.equiprop(h0, hs, values, dt, m_max=m)
    ref_seq, _, _ = oracle.equiprop(h0, hs, values, dt, m_max=m, reduction="sequential")
    ref_all, _, _ = oracle.equiprop_all(h0, hs, values, dt, m_max=m)
    tol, _ = parity_tolerance(ref, ref_seq, "fp64")
    ctx = sp.create(m_max=m)
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    amps = sp.ControlAmplitudes(values, dt)
    res = ctx.equiprop(amps)
    assert res.plan["m_max"] == m
    assert rel_fro(res.u, ref) <= tol
    cum = ctx.equiprop_all(amps)
    for k in (0, 1, 150, 299):
        assert rel_fro(cum.u_all[k], ref_all[k]) <= tol, k
    ctx.close()


@pytest.mark.parametrize("pts", [1000, 100_000, 1_000_000])
def test_driven_qubit_against_extended_precision_oracle(pts):
    """SURVEY.md §8(c) gate for d = 2: against the 80-bit oracle of the same
    midpoint discretisation (exact per-slice rotations, long double pairwise
    fold), the B200 result is at most twice as far off as the reference's
    own (oracle restatement, complex128)."""
    import oracle
    from cases import qubit_inputs
    h0, hs, values, dt = qubit_inputs(pts, "midpoint")
    exact = oracle.midpoint_reference_ld(1.0, 0.1, 1.0, 6.0, pts)
    ref, _, _ = oracle.equiprop(h0, hs, values, dt, mode="midpoint")
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    got = ctx.equiprop(sp.ControlAmplitudes(values, dt)).u
    err_ref = rel_fro(ref, exact)
    err_gpu = rel_fro(got, exact)
    assert err_gpu <= max(2.0 * err_ref, 1e-15), (err_gpu, err_ref)
    ctx.close()


@pytest.mark.parametrize("d", [2, 3, 4, 8, 16, 32])
def test_cumulative_complex64_against_oracle(d):
    """complex64 contexts (FP64 kernels, fp32 plan, complex64 output):
    the cumulative stack against the oracle's fp32 restatement within the
    complex64 gate, and the last entry equal to the sequential total."""
    import oracle
    from cases import random_inputs
    h0, hs, values, dt = random_inputs(d, 2, 300, 9100 + d)
    ref_all, _, _ = oracle.equiprop_all(h0, hs, values, dt, bits=32)
    ref, _, _ = oracle.equiprop(h0, hs, values, dt, bits=32)
    ref_seq, _, _ = oracle.equiprop(h0, hs, values, dt, bits=32, reduction="sequential")
    tol, _ = parity_tolerance(ref, ref_seq, "fp32")
    ctx = sp.create(precision="fp32")
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    amps = sp.ControlAmplitudes(values, dt)
    cum = ctx.equiprop_all(amps)
    assert cum.u_all.dtype == np.complex64 and cum.u_all.shape == ref_all.shape
    for k in (0, 1, 77, 150, 299):
        assert rel_fro(cum.u_all[k], ref_all[k]) <= tol, k
    assert np.array_equal(cum.final, ctx.equiprop(amps, reduction="sequential").u)
    ctx.close()
