"""GPU parity at the benchmarked scale: many slices per lane.

The lane kernels propagate a contiguous run of slices per warp / CTA / CTA
group through a pipelined loop (cross-step operand prefetch, next-slice
assembly during the series, ping-pong iterate buffers, group barriers, 3M
products whose rounding accumulates).  The golden cases are short (1-2
slices per lane on the wide families), so these tests run every family with
>= 32 slices per lane (asserted through ``ctx.last_lanes()``) against the CPU
oracle (bit-exact restatement of the reference) on the same seeded inputs,
and the headline C4 shape (d = 128, N = 4, midpoint) and its magnus variant
with >= 100 slices per lane.

Gate: rel-Frobenius <= max(1e-12, 4 eps_self), eps_self =
the reference's own pairwise-vs-sequential difference on the same input; the
measured error and eps_self are printed (run with -s).
"""

import functools

import numpy as np
import pytest

from cases import random_inputs
from helpers import parity_tolerance, rel_fro

import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def _reference(d, n_ctrl, pts, seed, mode):
    """Oracle pairwise and sequential totals from ONE slice-propagator batch."""
    import oracle
    h0, hs, values, dt = random_inputs(d, n_ctrl, pts, seed)
    u, _ = oracle.slice_propagators(h0, hs, values, dt, mode=mode)
    return oracle.reduce_pairwise(u), oracle.reduce_sequential(u), u.shape[0]


def _check(d, n_ctrl, pts, seed, mode, algo, min_per_lane):
    h0, hs, values, dt = random_inputs(d, n_ctrl, pts, seed)
    ref, ref_seq, count = _reference(d, n_ctrl, pts, seed, mode)
    tol, eps_self = parity_tolerance(ref, ref_seq, "fp64")
    with sp.create() as ctx:
        ctx.set_algorithm(algo)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        amps = sp.ControlAmplitudes(values, dt)
        res = ctx.equiprop(amps)
        lanes = ctx.last_lanes()
        kernel = ctx.last_timing()["kernel"]
        used = ctx.last_algorithm()["algorithm"]
        u_seq = ctx.equiprop(amps, reduction="sequential").u
    err = rel_fro(res.u, ref)
    err_seq = rel_fro(u_seq, ref)
    print(f"\n[scale parity] d={d} N={n_ctrl} {mode} slices={count} lanes={lanes} "
          f"({count / lanes:.0f}/lane) {kernel} {used}: err {err:.3e} seq {err_seq:.3e} "
          f"eps_self {eps_self:.3e} tol {tol:.3e}")
    assert res.slice_count == count
    assert count / lanes >= min_per_lane, (count, lanes)
    assert err <= tol, (err, tol, eps_self)
    assert err_seq <= tol, (err_seq, tol, eps_self)


@pytest.mark.parametrize("algo", ["auto", "ps", "clenshaw"])
def test_c4_shape_many_slices_per_lane(algo):
    """C4 shape (d = 128, N = 4, midpoint, beta = 0.5, m = 13): 37 lanes x
    110 slices through the pipelined group loop."""
    _check(128, 4, 37 * 110, 20240911, "midpoint", algo, 100)


def test_c4_magnus_many_slices_per_lane():
    """C4 magnus variant (T = 15 terms, m = 15): pts = 2 * 37 * 108 + 1."""
    _check(128, 4, 2 * 37 * 108 + 1, 20240912, "magnus", "auto", 100)


@pytest.mark.parametrize("algo", ["auto", "ps", "ps3m"])
@pytest.mark.parametrize("d,n_ctrl,pts,mode", [
    (64, 2, 40 * 148, "midpoint"),
    (96, 3, 2 * 40 * 37 + 1, "simpson"),
    (200, 2, 36 * 9, "midpoint"),
    (512, 2, 34 * 2, "midpoint"),
])
def test_group_families_many_slices_per_lane(d, n_ctrl, pts, mode, algo):
    """D64 / D128 / D256 / D512 group kernels with >= 32 slices per lane."""
    _check(d, n_ctrl, pts, 31 * d + n_ctrl, mode, algo, 32)


@pytest.mark.parametrize("d", [8, 16, 32])
def test_warp_and_cta_families_many_slices_per_lane(d):
    """D8 (warp lanes), D16 (4 lanes per CTA), D32 (CTA lanes) with >= 32
    slices per lane."""
    lanes_cap = {8: 148 * 3 * 8, 16: 148 * 2 * 4, 32: 148 * 2}[d]
    _check(d, 2, 34 * lanes_cap, 77 + d, "midpoint", "auto", 32)


def test_c3_random_1e5_slices():
    """C3 shape (d = 32, N = 2, m = 13) at 1e5 slices."""
    _check(32, 2, 100_000, 20240911, "midpoint", "auto", 32)
