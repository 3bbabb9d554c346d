"""Driven-qubit error of the B200 path and of the reference restatement against
the 80-bit oracle of the same midpoint discretisation.

    python tools/qubit_ld_err.py
"""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests'); sys.path.insert(0,'tests/golden')
import oracle, paper_2108_07126_b200 as sp
from cases import qubit_inputs
from helpers import rel_fro
for pts in (1000, 100000, 1000000, 10000000):
    h0, hs, values, dt = qubit_inputs(pts, "midpoint")
    exact = oracle.midpoint_reference_ld(1.0, 0.1, 1.0, 6.0, pts)
    ref, _, _ = oracle.equiprop(h0, hs, values, dt, mode="midpoint") if pts <= 1000000 else (None,0,0)
    ctx = sp.create(); ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    got = ctx.equiprop(sp.ControlAmplitudes(values, dt)).u
    print(pts, "err_gpu %.3e" % rel_fro(got, exact), "err_ref %s" % ("%.3e" % rel_fro(ref, exact) if ref is not None else "-"), flush=True)
