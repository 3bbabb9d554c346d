import sys, json, statistics
sys.path[:0] = ['tests/golden', '.']
import torch, paper_2108_07126_b200 as sp
from cases import qubit_inputs
n = 4_000_000
h0, hs, v, dt = qubit_inputs(n, 'midpoint')
ctx = sp.create(); ctx.set_hamiltonian(sp.ControlSystem(h0, hs)); plan = ctx.plan_for(dt)
d = torch.from_numpy(v).cuda(); o = torch.empty((2, 2), dtype=torch.complex128, device='cuda')
oa = torch.empty((n, 2, 2), dtype=torch.complex128, device='cuda')
st = torch.cuda.current_stream()
res = {}
for name, fn in (("pairwise", lambda: ctx.equiprop_device_ptr(d.data_ptr(), n, 2, dt, o.data_ptr(), stream=st.cuda_stream, plan=plan)),
                 ("sequential", lambda: ctx.equiprop_device_ptr(d.data_ptr(), n, 2, dt, o.data_ptr(), stream=st.cuda_stream, plan=plan, reduction="sequential")),
                 ("all", lambda: ctx.equiprop_all_device_ptr(d.data_ptr(), n, 2, dt, oa.data_ptr(), stream=st.cuda_stream, plan=plan))):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    res[name] = (round(statistics.median(ts), 4), ctx.last_timing()["kernel"])
print(json.dumps(res))
