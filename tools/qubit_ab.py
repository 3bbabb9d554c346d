"""A/B timing of the d = 2 lane kernel across library builds.

    python tools/qubit_ab.py LIB1.so LIB2.so ...

Each library runs in its own process (SLICEPROP_B200_LIB): driven qubit at
1e5 / 1e6 slices and a random d = 2 system (m = 13) at 1e6, best of 20
kernel times (CUDA events inside the library) and the end-to-end call.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, json
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests/golden")
import numpy as np
import paper_2108_07126_b200 as sp
from cases import random_inputs, qubit_inputs
out = {}
for label, args in (("qubit 1e5", qubit_inputs(100000, "midpoint")),
                    ("qubit 1e6", qubit_inputs(1000000, "midpoint")),
                    ("rand d2 1e6", random_inputs(2, 2, 1000000, 1))):
    h0, hs, v, dt = args
    ctx = sp.create(); ctx.set_hamiltonian(sp.ControlSystem(h0, hs)); ctx.set_profiling(True)
    r = ctx.equiprop(sp.ControlAmplitudes(v, dt))
    best = 1e9
    for _ in range(20):
        ctx.equiprop(sp.ControlAmplitudes(v, dt)); best = min(best, ctx.last_timing()["main_kernel_ms"])
    out[label] = dict(us=round(best * 1e3, 2), kernel=ctx.last_timing()["kernel"],
                      u00=repr(complex(r.u[0, 0])))
    ctx.close()
print(json.dumps(out))
'''.replace("ROOT", repr(ROOT))
for lib in sys.argv[1:]:
    env = dict(os.environ, SLICEPROP_B200_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(lib, r.stdout.strip() or r.stderr[-800:], flush=True)
