"""One propagation of a bench workload at a chosen slice count (ncu target).

    python tools/ncu_target.py --workload c4 --slices 2000 [--repeat 2]
"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
import paper_2108_07126_b200 as sp

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c4")
ap.add_argument("--slices", type=int, default=2000)
ap.add_argument("--repeat", type=int, default=2)
a = ap.parse_args()
wl = dict(bench.WORKLOADS[a.workload]); wl["slices"] = a.slices
h0, hs, values, dt = bench.make_problem(wl)
ctx = sp.create()
ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=wl["mode"] == "magnus",
                    quadrature=None if wl["mode"] == "magnus" else wl["mode"])
amps = sp.ControlAmplitudes(values, dt)
for _ in range(a.repeat):
    u = ctx.equiprop(amps).u
print("done", a.workload, a.slices, np.linalg.norm(u))
