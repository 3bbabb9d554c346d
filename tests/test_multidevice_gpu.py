"""Single-process multi-device contexts (``create(devices=[...])`` /
``sp_create(ctx, bits, num_gpus, device_ids)``).

The box has one B200, so the P devices are emulated by repeating ordinal 0:
every block still runs on its own child context and stream, the block
products are gathered by (same-device) peer copies and multiplied in time
order — the code path a P-GPU host runs, minus NVLink.  Results must equal
the single-device propagation within the parity gate (matrix products are
associative; only the association changes) and the oracle on the same
inputs; amplitude violations report the GLOBAL first offender.
"""

import numpy as np
import pytest

from cases import qubit_inputs, random_inputs
from helpers import parity_tolerance, rel_fro

import paper_2108_07126_b200 as sp

pytestmark = pytest.mark.gpu


def _pair(h0, hs, values, dt, mode, precision, devices, reduction="pairwise"):
    out = []
    for devs in (None, devices):
        ctx = sp.create(precision=precision, devices=devs)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        res = ctx.equiprop(sp.ControlAmplitudes(values, dt), reduction=reduction)
        out.append(res)
        ctx.close()
    return out


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("reduction", ["pairwise", "sequential"])
@pytest.mark.parametrize("d,mode,pts", [(2, "midpoint", 4001), (2, "magnus", 2001),
                                        (8, "simpson", 801), (32, "midpoint", 600),
                                        (128, "midpoint", 300), (64, "magnus", 201)])
def test_emulated_devices_match_single_device_and_oracle(d, mode, pts, reduction, precision):
    import oracle
    h0, hs, values, dt = random_inputs(d, 2, pts, 300 + d)
    single, multi = _pair(h0, hs, values, dt, mode, precision, [0, 0, 0, 0], reduction)
    bits = 32 if precision == "fp32" else 64
    ref, n, _ = oracle.equiprop(h0, hs, values, dt, mode=mode, bits=bits)
    ref_seq, _, _ = oracle.equiprop(h0, hs, values, dt, mode=mode, bits=bits,
                                    reduction="sequential")
    tol, eps = parity_tolerance(ref, ref_seq, precision)
    assert multi.slice_count == single.slice_count == n
    assert multi.u.dtype == single.u.dtype == ref.dtype
    assert multi.plan == single.plan
    assert rel_fro(multi.u, single.u) <= tol
    err = rel_fro(multi.u, ref)
    if precision == "fp32" and d > 8 and err > tol:
        # d >= 9 complex64 contexts compute in FP64 and round: where they
        # leave the complex64 gate it is because the reference's own
        # complex64 result is further from the exact (complex128) one
        ref64, _, _ = oracle.equiprop(h0, hs, values, dt, mode=mode, bits=64)
        assert rel_fro(multi.u, ref64) <= rel_fro(ref, ref64), (err, tol, eps)
    else:
        assert err <= tol, (err, tol, eps)


def test_more_devices_than_slices_and_empty_table():
    h0, hs, values, dt = qubit_inputs(3, "midpoint")
    single, multi = _pair(h0, hs, values, dt, "midpoint", "fp64", [0] * 5)
    assert rel_fro(multi.u, single.u) <= 1e-15
    ctx = sp.create(devices=[0, 0])
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    res = ctx.equiprop(sp.ControlAmplitudes(np.zeros((0, 2)), dt))
    assert res.slice_count == 0 and np.array_equal(res.u, np.eye(2))
    ctx.close()


@pytest.mark.parametrize("mode", ["midpoint", "simpson"])
def test_global_first_amplitude_violation(mode):
    """Offenders in blocks 1 and 3 of 4: the error names the row-major
    first one over the WHOLE table, with the reference's message
    (hamiltonian.py:170-174), exactly as the single-device call does."""
    h0, hs, values, dt = random_inputs(4, 2, 401, 17)
    values = values.copy()
    values[150, 1] = 1.5    # block 1 (of 4 x 50 slices: rows 100..200)
    values[380, 0] = -2.0   # block 3
    msgs = []
    for devs in (None, [0, 0, 0, 0]):
        ctx = sp.create(devices=devs)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs),
                            quadrature=None if mode == "midpoint" else mode)
        with pytest.raises(sp.AmplitudeBoundError) as exc:
            ctx.equiprop(sp.ControlAmplitudes(values, dt, copy=False))
        msgs.append(str(exc.value))
        ctx.close()
    assert msgs[0] == msgs[1]
    assert "sample 150, control 1" in msgs[1]


def test_device_entry_points_run_on_first_device():
    """equiprop_all and the device-resident entry of a multi-device context
    run on devices[0] and equal the single-device results bit for bit."""
    h0, hs, values, dt = random_inputs(8, 2, 257, 5)
    amps = sp.ControlAmplitudes(values, dt)
    a = sp.create()
    a.set_hamiltonian(sp.ControlSystem(h0, hs))
    b = sp.create(devices=[0, 0, 0])
    b.set_hamiltonian(sp.ControlSystem(h0, hs))
    assert np.array_equal(a.equiprop_all(amps).u_all, b.equiprop_all(amps).u_all)
    a.close()
    b.close()
