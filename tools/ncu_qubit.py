"""Driven-qubit propagation (C1 system) at a chosen slice count (ncu target).

    python tools/ncu_qubit.py SLICES
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_07126_b200 as sp  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
q = sp.DrivenQubit(1.0, 0.1, 1.0, 6.0)
ctx = sp.create()
ctx.set_hamiltonian(q.system())
print(ctx.equiprop(q.amplitudes(n)).u)
