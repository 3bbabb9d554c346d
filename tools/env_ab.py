"""A/B kernel timing of random systems under environment variants.

    python tools/env_ab.py "d,n_ctrl,slices,prec[,algo[,mode]];..." "" "SP_D64_GROUP=2" ...

Each variant (space-separated VAR=VALUE list; "" = defaults) runs in its own
process; per case: kernel name, best of 10 main-kernel times (CUDA events in
the library), executed-FP64 fraction of the measured DMMA peak, and U[0,0].
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
    mode = rest[1] if len(rest) > 1 else "midpoint"
    pts = int(n) if mode == "midpoint" else 2 * int(n) + 1
    h0, hs, v, dt = random_inputs(int(d), int(nc), pts, 1)
    ctx = sp.create(precision=prec)
    if rest and rest[0] != "auto":
        ctx.set_algorithm(rest[0])
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    ctx.set_profiling(True)
    amps = sp.ControlAmplitudes(v, dt)
    r = ctx.equiprop(amps)
    best, flops = 1e9, 0.0
    for _ in range(10):
        ctx.equiprop(amps)
        t = ctx.last_timing()
        if t["main_kernel_ms"] < best:
            best, flops = t["main_kernel_ms"], t["executed_flops"]
    out[case] = dict(kernel=t["kernel"], ms=round(best, 4), lanes=ctx.last_lanes(),
                     exec_frac=round(flops / (best / 1e3) / 37.09e12, 3),
                     u00=repr(complex(r.u[0, 0])))
    ctx.close()
print(json.dumps(out))
'''


def main():
    cases, variants = sys.argv[1], sys.argv[2:] or [""]
    child = CHILD.replace("ROOT", repr(ROOT)).replace("CASES", repr(cases))
    for variant in variants:
        env = dict(os.environ)
        for kv in variant.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True,
                           text=True, cwd=ROOT)
        print(f"[{variant or 'default'}]", r.stdout.strip() or r.stderr[-1500:], flush=True)


if __name__ == "__main__":
    main()
