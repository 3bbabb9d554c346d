"""A/B kernel timing of random systems across library builds.

    python tools/dim_ab.py "d,n_ctrl,slices,prec[,algo];..." LIB1.so LIB2.so ...

Each library runs in its own process (SLICEPROP_B200_LIB); best of 10
kernel times (CUDA events inside the library) per case, and the first
element of the result to compare numerics.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests/golden")
import paper_2108_07126_b200 as sp
from cases import random_inputs
out = {}
for case in CASES.split(";"):
    d, nc, n, prec, *rest = case.split(",")
    h0, hs, v, dt = random_inputs(int(d), int(nc), int(n), 1)
    ctx = sp.create(precision=prec)
    if rest:
        ctx.set_algorithm(rest[0])
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs)); ctx.set_profiling(True)
    amps = sp.ControlAmplitudes(v, dt)
    r = ctx.equiprop(amps)
    best = 1e9
    for _ in range(10):
        ctx.equiprop(amps); best = min(best, ctx.last_timing()["main_kernel_ms"])
    out[case] = dict(us=round(best * 1e3, 2), kernel=ctx.last_timing()["kernel"], u00=repr(complex(r.u[0, 0])))
    ctx.close()
print(json.dumps(out))
'''.replace("ROOT", repr(ROOT))
cases = sys.argv[1]
for lib in sys.argv[2:]:
    env = dict(os.environ, SLICEPROP_B200_LIB=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", CHILD.replace("CASES", repr(cases))], env=env,
                       capture_output=True, text=True)
    print(lib, r.stdout.strip() or r.stderr[-800:], flush=True)
