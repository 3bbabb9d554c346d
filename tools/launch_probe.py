"""Small-n launches for an ncu duration comparison (ncu target).

    ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg python tools/launch_probe.py N

Runs, in order: a trivial torch kernel (zero_ of 4 floats), the driven qubit
at N slices through the default path, then the same through the cp.async su2
form (SP_SU2_TMA=0) and the general d = 2 kernel (SP_SU2=0), each in a child
process so the environment switches take effect.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000
child = (f"import sys; sys.path[:0] = [{ROOT!r}, {ROOT + '/tests/golden'!r}];"
         "import torch, paper_2108_07126_b200 as sp; from cases import qubit_inputs;"
         f"h0, hs, v, dt = qubit_inputs({n}, 'midpoint'); ctx = sp.create();"
         "ctx.set_hamiltonian(sp.ControlSystem(h0, hs));"
         "[ctx.equiprop(sp.ControlAmplitudes(v, dt)) for _ in range(2)];"
         "print(ctx.last_timing()['kernel'])")
import torch  # noqa: E402

o = torch.empty(4, device="cuda")
for _ in range(2):
    o.zero_()
torch.cuda.synchronize()
for env in ({}, {"SP_SU2_TMA": "0"}, {"SP_SU2": "0"}):
    subprocess.run([sys.executable, "-c", child], env=dict(os.environ, **env), check=True)
