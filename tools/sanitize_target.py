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

# SANITIZE_NO_TMEM=1: skip the kernels that use tensor memory (tcgen05
# alloc/ld/st: the ps3 / ps3g families), for tools that do not model it
NO_TMEM = os.environ.get("SANITIZE_NO_TMEM") == "1"

for d, n in ((2, 300), (3, 40), (4, 64), (8, 40), (16, 16), (32, 8), (64, 6), (128, 3),
             (256, 2), (512, 2)):
    for algo in ("clenshaw", "ps", "ps3m") if 16 <= d <= 256 else ("auto",):
        if NO_TMEM and (algo == "ps3m" or (algo == "auto" and d >= 64)):
            continue
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
