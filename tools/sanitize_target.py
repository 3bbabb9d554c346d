"""Small propagations through every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_target.py
    compute-sanitizer --tool racecheck python tools/sanitize_target.py
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests", "golden"))
import numpy as np
import paper_2108_07126_b200 as sp
from cases import random_inputs

for d, n in ((2, 300), (4, 64), (16, 16), (32, 8), (64, 6), (128, 3), (256, 2)):
    for algo in ("clenshaw", "ps", "ps3m") if d >= 16 else ("auto",):
        h0, hs, v, dt = random_inputs(d, 2, n, 7)
        ctx = sp.create()
        ctx.set_algorithm(algo)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        amps = sp.ControlAmplitudes(v, dt)
        u = ctx.equiprop(amps).u
        useq = ctx.equiprop(amps, reduction="sequential").u
        cum = ctx.equiprop_all(amps)
        assert np.array_equal(cum.final, useq)
        print(f"d={d} {algo}: unitarity {np.abs(u.conj().T @ u - np.eye(d)).max():.2e}", flush=True)
        ctx.close()
print("sanitize target done")
