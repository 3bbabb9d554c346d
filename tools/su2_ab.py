"""A/B timing of the d = 2 driven-qubit step under environment variants.

    python tools/su2_ab.py [--slices 1e5,1e6,1e7] "SP_SU2=0" "SP_SU2_TPB=512" ...

Each variant (space-separated VAR=VALUE list; "" = defaults) runs in its own
process.  Timing as bench.py times C1/c1m: the step captured in a CUDA graph,
L2 flushed (256 MiB write) before every replay, CUDA events around the
replay on the launching stream; median and best of 30 replays.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, statistics
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests/golden")
import numpy as np, torch
import paper_2108_07126_b200 as sp
from cases import qubit_inputs
out = {}
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
def l2_flush(k):
    flush.fill_(float(k)); clean.sum()  # write, then read: L2 left clean and cold
for n in SLICES:
    h0, hs, v, dt = qubit_inputs(n, "midpoint")
    ctx = sp.create(); ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    plan = ctx.plan_for(dt)
    d = torch.from_numpy(v).cuda(); o = torch.empty((2, 2), dtype=torch.complex128, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            ctx.equiprop_device_ptr(d.data_ptr(), n, 2, dt, o.data_ptr(), stream=st.cuda_stream, plan=plan)
    torch.cuda.synchronize()
    kernel = ctx.last_timing()["kernel"]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        ctx.equiprop_device_ptr(d.data_ptr(), n, 2, dt, o.data_ptr(), stream=st.cuda_stream, plan=plan)
    ts = []
    with torch.cuda.stream(st):
        for k in range(33):
            l2_flush(k)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st); g.replay(); b.record(st); st.synchronize()
            if k >= 3: ts.append(a.elapsed_time(b) * 1e3)
    ref = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u
    tn = []
    with torch.cuda.stream(st):
        for k in range(33):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st); g.replay(); b.record(st); st.synchronize()
            if k >= 3: tn.append(a.elapsed_time(b) * 1e3)
    out[f"{n:.0e}"] = dict(med_us=round(statistics.median(ts), 2), best_us=round(min(ts), 2),
                          noflush_med_us=round(statistics.median(tn), 2),
                          kernel=kernel, lanes=ctx.last_lanes(), u00=repr(complex(ref[0, 0])))
    ctx.close()
# floors: the same protocol around one trivial kernel, as a graph / a direct
# launch, with / without the L2 flush in front
o = torch.empty(4, device="cuda"); st = torch.cuda.Stream(); g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    o.zero_()
for name, use_graph, do_flush in (("graph_flush", 1, 1), ("graph_noflush", 1, 0),
                                  ("direct_flush", 0, 1), ("direct_noflush", 0, 0)):
    ts = []
    with torch.cuda.stream(st):
        for k in range(33):
            if do_flush: l2_flush(k)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(st)
            if use_graph: g.replay()
            else: o.zero_()
            b.record(st); st.synchronize()
            if k >= 3: ts.append(a.elapsed_time(b) * 1e3)
    out["floor_" + name] = round(statistics.median(ts), 2)
print(json.dumps(out))
'''


def main():
    args = sys.argv[1:]
    slices = [100_000, 1_000_000, 10_000_000]
    if args and args[0] == "--slices":
        slices = [int(float(x)) for x in args[1].split(",")]
        args = args[2:]
    child = CHILD.replace("ROOT", repr(ROOT)).replace("SLICES", repr(slices))
    for variant in args or [""]:
        env = dict(os.environ)
        for kv in variant.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True,
                           text=True, cwd=ROOT)
        print(f"[{variant or 'default'}]", r.stdout.strip() or r.stderr[-1500:], flush=True)


if __name__ == "__main__":
    main()
