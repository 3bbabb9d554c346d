"""One propagation of a random system (ncu target).

    python tools/env_ab_target.py D N_CTRL SLICES [fp64|fp32]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]
import paper_2108_07126_b200 as sp  # noqa: E402
from cases import random_inputs  # noqa: E402

d, nc, n = (int(x) for x in sys.argv[1:4])
prec = sys.argv[4] if len(sys.argv) > 4 else "fp64"
h0, hs, v, dt = random_inputs(d, nc, n, 1)
ctx = sp.create(prec)
ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
print(ctx.equiprop(sp.ControlAmplitudes(v, dt)).u[0, 0], ctx.last_timing()["kernel"])
