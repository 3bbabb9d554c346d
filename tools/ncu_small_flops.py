"""ncu target for the executed-FP64 model of the register families
(lane_small_kernel<2,1> / <4,4>): one propagation per (d, m, N) point on
random systems with m pinned, 2^20 slices each (run under
`ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on.sum`).

    python tools/ncu_small_flops.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2108_07126_b200 as sp  # noqa: E402
from cases import qubit_inputs, random_inputs  # noqa: E402

N = 1 << 20
POINTS = [("qubit", 2, 2, 3)] + [("rand", 2, 2, m) for m in (3, 7, 13, 15, 5)] + \
         [("rand", 2, 1, 13), ("rand", 2, 4, 13)] + \
         [("rand", 4, 2, m) for m in (3, 7, 13, 25)] + [("rand", 3, 2, 13), ("rand", 4, 4, 13)]
for kind, d, n_ctrl, m in POINTS:
    if kind == "qubit":
        h0, hs, v, dt = qubit_inputs(N, "midpoint")
    else:
        h0, hs, v, dt = random_inputs(d, n_ctrl, N, 11 + d + m, beta=0.1)
    with sp.create(m_max=m) as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        u = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u
        print(kind, d, n_ctrl, m, ctx.last_timing()["kernel"], ctx.last_lanes(), float(np.abs(u).sum()),
              flush=True)
# complex-pair (generic) d = 2 path: more controls, three-point modes
for mode, n_ctrl, m in (("midpoint", 3, 13), ("midpoint", 4, 3), ("midpoint", 4, 7),
                        ("simpson", 2, 13), ("magnus", 2, 13)):
    pts = N if mode == "midpoint" else 2 * N + 1
    h0, hs, v, dt = random_inputs(2, n_ctrl, pts, 5 + n_ctrl + m, beta=0.1)
    with sp.create(m_max=m) as ctx:
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                            quadrature=None if mode == "magnus" else mode)
        u = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u
        print(mode, 2, n_ctrl, m, ctx.last_timing()["kernel"], float(np.abs(u).sum()), flush=True)
