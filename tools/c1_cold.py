"""Where the C1 / north-star qubit step time goes: the same graph-replayed
launch timed (a) back to back, (b) after a 256 MiB L2 flush (bench protocol),
(c) after a flush of only 32 MiB (L2 still holds the kernel code and params).

    python tools/c1_cold.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2108_07126_b200 as sp  # noqa: E402
from cases import qubit_inputs  # noqa: E402

dev = torch.device("cuda", 0)
for n in (100000, 1000000):
    h0, hs, v, dt = qubit_inputs(n, "midpoint")
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    plan = ctx.plan_for(dt)
    d_amps = torch.from_numpy(np.ascontiguousarray(v)).to(dev)
    out = torch.empty((2, 2), dtype=torch.complex128, device=dev)
    big = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    small = torch.empty(8 * 1024 * 1024, dtype=torch.float32, device=dev)
    s = torch.cuda.Stream(dev)
    ctx.set_profiling(False)
    for _ in range(3):
        ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(), stream=s.cuda_stream, plan=plan)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(), stream=s.cuda_stream, plan=plan)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream(dev)
    g20 = torch.cuda.CUDAGraph()  # 20 launches per replay: not host-bound
    with torch.cuda.graph(g20, stream=s):
        for _ in range(20):
            ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                    stream=s.cuda_stream, plan=plan)
    g20.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for _ in range(10):
        g20.replay()
    e1.record(cur)
    torch.cuda.synchronize()
    b2b = e0.elapsed_time(e1) / 200 * 1e3
    res = {}
    for name, buf in (("flush256", big), ("flush32", small), ("none", None)):
        ts = []
        for k in range(30):
            if buf is not None:
                buf.fill_(float(k))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(cur)
            g.replay()
            b.record(cur)
            cur.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        res[name] = float(np.median(ts))
    ts = []
    for k in range(30):  # direct launch (no graph) after the 256 MiB flush
        big.fill_(float(k))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                stream=cur.cuda_stream, plan=plan)
        b.record(cur)
        cur.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    res["direct"] = float(np.median(ts))
    print(f"n={n}: back-to-back {b2b:.2f} us/step; single replay after flush 256 MiB "
          f"{res['flush256']:.2f}, after 32 MiB {res['flush32']:.2f}, no flush {res['none']:.2f} us; direct launch after 256 MiB {res['direct']:.2f} us",
          flush=True)
    ctx.close()
