"""One random-system propagation at a chosen dimension (ncu target).

    python tools/ncu_dim.py D N_CTRL SLICES [algo]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests", "golden"))
import paper_2108_07126_b200 as sp  # noqa: E402
from cases import random_inputs  # noqa: E402

d, nc, n = (int(x) for x in sys.argv[1:4])
algo = sys.argv[4] if len(sys.argv) > 4 else "auto"
h0, hs, v, dt = random_inputs(d, nc, n, 1)
ctx = sp.create()
ctx.set_algorithm(algo)
ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
print(ctx.equiprop(sp.ControlAmplitudes(v, dt)).u[0, 0])
