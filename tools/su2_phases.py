"""Phase timestamps of the su(2) kernel (SP_SU2_PROF=1 build hook): for each
slice count, 5 cold calls (L2 written then read between calls), the library
prints min / max over CTAs of %globaltimer at kernel entry (p0), first row
stage landed (p1), lane loop done (p2), CTA product (p3), last CTA's ticket
(p4) and result written (p5), in ns from the first CTA's entry.

    SP_SU2_PROF=1 python tools/su2_phases.py 1000 100000 1000000
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests", "golden")]
os.environ.setdefault("SP_SU2_PROF", "1")
import torch  # noqa: E402

import paper_2108_07126_b200 as sp  # noqa: E402
from cases import qubit_inputs  # noqa: E402

flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for n in [int(float(a)) for a in sys.argv[1:]] or [1000, 100000, 1000000]:
    h0, hs, v, dt = qubit_inputs(n, "midpoint")
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
    plan = ctx.plan_for(dt)
    d = torch.from_numpy(v).cuda()
    o = torch.empty((2, 2), dtype=torch.complex128, device="cuda")
    for k in range(6):
        flush.fill_(float(k))
        clean.sum()
        torch.cuda.synchronize()
        ctx.equiprop_device_ptr(d.data_ptr(), n, 2, dt, o.data_ptr(), plan=plan)
        torch.cuda.synchronize()
    ctx.close()
