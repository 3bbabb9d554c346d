"""Scaling and squaring past the series capability (north-star extension N1,
paper_2108_07126_b200/scaling.py).

The reference raises StepTooLargeError above the m = 25 capability
(chebyshev.py:113-134) and so does a default context.  With scaling=True the
step is propagated through per-slice norm bounds, a reduced-bound Chebyshev
plan and s batched squarings on the device.  There is no reference output
for such steps, so the gate is an independent oracle: exact per-slice
exponentials exp(-i G_k) by eigendecomposition of the (Hermitian) exponents,
multiplied in time order in complex128 — rel-Frobenius <= 1e-11 (complex128;
the squarings amplify the series rounding by ~2^s) and 2e-5 (complex64).
"""

import numpy as np
import pytest

from helpers import rel_fro

import paper_2108_07126_b200 as sp
from paper_2108_07126_b200.scaling import slice_table

pytestmark = pytest.mark.gpu


def unit_hermitian(rng, d):
    a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    h = 0.5 * (a + a.conj().T)
    return h / np.abs(h).sum(axis=0).max()


def eig_oracle(ctx, amps):
    """exp(-i G_k) by eigh, ordered product (later on the left)."""
    terms = ctx._effective.terms() if ctx._magnus else ctx._system.terms()
    table, scale = slice_table(ctx, amps)
    stack = np.stack(terms)
    u = np.eye(stack.shape[1], dtype=complex)
    for row in table:
        g = scale * np.tensordot(row, stack, axes=1)
        g = 0.5 * (g + g.conj().T)
        w, v = np.linalg.eigh(g)
        u = (v * np.exp(-1j * w)) @ v.conj().T @ u
    return u


def make(d, n_ctrl, pts, beta, seed, mode="midpoint", precision="fp64"):
    rng = np.random.default_rng(seed)
    h0 = unit_hermitian(rng, d)
    hs = [unit_hermitian(rng, d) for _ in range(n_ctrl)]
    step_scale = 1.0 if mode == "midpoint" else 2.0
    dt = beta / (step_scale * (n_ctrl + 1))
    values = rng.uniform(-1.0, 1.0, (pts, n_ctrl))
    ctx = sp.create(precision, scaling=True)
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    return ctx, sp.ControlAmplitudes(values, dt)


@pytest.mark.parametrize("d", [2, 3, 8, 33, 64, 128])
def test_beyond_capability_matches_eigen_oracle(d):
    ctx, amps = make(d, 2, 301 if d < 64 else 61, 20.0, 100 + d)
    res = ctx.equiprop(amps)
    ref = eig_oracle(ctx, amps)
    err = rel_fro(res.u, ref)
    print(f"\n[scaling] d={d} beta={res.plan['beta']:.1f} m={res.plan['m_max']} "
          f"s={res.plan['squarings']}: rel err {err:.3e}")
    assert res.plan["beta"] > 4.447 and res.plan["squarings"] >= 1
    assert err <= 1e-11
    ctx.close()


@pytest.mark.parametrize("mode", ["simpson", "magnus"])
def test_three_point_modes(mode):
    ctx, amps = make(8, 2, 2 * 150 + 1, 12.0, 7, mode=mode)
    res = ctx.equiprop(amps)
    err = rel_fro(res.u, eig_oracle(ctx, amps))
    print(f"\n[scaling] {mode}: s={res.plan['squarings']} rel err {err:.3e}")
    assert err <= 1e-11
    assert rel_fro(ctx.equiprop(amps, reduction="sequential").u, res.u) <= 1e-12
    ctx.close()


def test_chunked_product(monkeypatch):
    """Many chunks (CHUNK_BYTES shrunk to 64 KiB: 16 slices of d = 16 per
    chunk) give the same propagator as the oracle."""
    import paper_2108_07126_b200.scaling as scaling
    monkeypatch.setattr(scaling, "CHUNK_BYTES", 64 << 10)
    ctx, amps = make(16, 1, 2000, 20.0, 11)
    res = ctx.equiprop(amps)
    err = rel_fro(res.u, eig_oracle(ctx, amps))
    print(f"\n[scaling] 125 chunks d=16: rel err {err:.3e}")
    assert err <= 1e-11
    ctx.close()


def test_fp32():
    """complex64 context past its capability (9.919): complex64 arithmetic,
    per-slice error ~ u32 * beta amplified by the squarings, summed over the
    slices: gate 2e-4 at 200 slices (the oracle is complex128)."""
    ctx, amps = make(16, 1, 200, 30.0, 11, precision="fp32")
    res = ctx.equiprop(amps)
    assert res.u.dtype == np.complex64
    err = rel_fro(res.u, eig_oracle(ctx, amps))
    print(f"\n[scaling] fp32 d=16 beta=30 (capability 9.919) m={res.plan['m_max']} "
          f"s={res.plan['squarings']}: rel err {err:.3e}")
    assert res.plan["squarings"] >= 1
    assert err <= 2e-4
    ctx.close()


def test_default_context_still_raises_and_within_capability_is_unchanged():
    rng = np.random.default_rng(3)
    h0, hs = unit_hermitian(rng, 8), [unit_hermitian(rng, 8)]
    values = rng.uniform(-1, 1, (100, 1))
    with sp.create() as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        with pytest.raises(sp.StepTooLargeError):
            ctx.equiprop(sp.ControlAmplitudes(values, 10.0))
        u_plain = ctx.equiprop(sp.ControlAmplitudes(values, 0.2)).u
        ctx.set_scaling(True)
        assert np.array_equal(ctx.equiprop(sp.ControlAmplitudes(values, 0.2)).u, u_plain)
        big = ctx.equiprop(sp.ControlAmplitudes(values, 10.0))
        assert big.plan["squarings"] >= 1
        bad = values.copy()
        bad[7, 0] = 1.5
        with pytest.raises(sp.AmplitudeBoundError, match="sample 7, control 0"):
            ctx.equiprop(sp.ControlAmplitudes(bad, 10.0))


def test_cli_and_binding_expose_scaling(tmp_path):
    """`propagate --scaling` and pysliceprop.Session(scaling=True) reach the
    extension; without them the reference's StepTooLargeError (CLI exit 3)."""
    import json
    import subprocess
    import sys
    from paper_2108_07126_b200 import pysliceprop
    rng = np.random.default_rng(8)
    h0, h1 = unit_hermitian(rng, 4), unit_hermitian(rng, 4)
    values = rng.uniform(-1, 1, (50, 1))
    pairs = lambda m: np.stack([m.real, m.imag], axis=-1).tolist()
    manifest = {"dim": 4, "drift": pairs(h0), "controls": [pairs(h1)], "dt": 6.0,
                "amplitudes": {"pts": 50, "data": values.tolist()}}
    path = tmp_path / "m.json"
    path.write_text(json.dumps(manifest))
    root = __import__("os").path.dirname(__import__("os").path.dirname(__file__))
    base = [sys.executable, "-m", "paper_2108_07126_b200", "propagate", str(path)]
    r = subprocess.run(base, cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 3, r.stderr
    r = subprocess.run(base + ["--scaling"], cwd=root, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert "squarings" in r.stderr
    u_cli = np.array(json.loads(r.stdout)["u"])
    with pysliceprop.Session(scaling=True) as s:
        s.set_hamiltonian(h0, [h1])
        u = s.equiprop(values, 6.0)
    assert np.allclose(u_cli[..., 0] + 1j * u_cli[..., 1], u, rtol=0, atol=1e-12)
