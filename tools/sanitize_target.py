"""Small propagations through every kernel family, for compute-sanitizer:

    compute-sanitizer --tool memcheck  python tools/sanitize_target.py
    compute-sanitizer --tool racecheck python tools/sanitize_target.py
"""
import os, sys
os.environ.setdefault("SP_F32_REG2", "1")  # the d = 2 register lanes at any size
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests", "golden"))
import numpy as np
import paper_2108_07126_b200 as sp
from cases import random_inputs

# SANITIZE_NO_TMEM=1: skip the kernels that use tensor memory (tcgen05
# alloc/ld/st: the ps3 / ps3g families), for tools that do not model it
NO_TMEM = os.environ.get("SANITIZE_NO_TMEM") == "1"

for d, n in ((2, 300), (3, 40), (4, 64), (8, 40), (16, 16), (32, 8), (64, 6), (128, 3),
             (256, 2), (512, 2)):
    for algo in ("clenshaw", "ps", "ps3m") if 16 <= d <= 256 else ("auto",):
        if NO_TMEM and (algo == "ps3m" or (algo == "auto" and d >= 64)):
            continue
        h0, hs, v, dt = random_inputs(d, 2, n, 7)
        ctx = sp.create()
        ctx.set_algorithm(algo)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        amps = sp.ControlAmplitudes(v, dt)
        u = ctx.equiprop(amps).u
        useq = ctx.equiprop(amps, reduction="sequential").u
        cum = ctx.equiprop_all(amps)
        assert np.array_equal(cum.final, useq)
        print(f"d={d} {algo}: unitarity {np.abs(u.conj().T @ u - np.eye(d)).max():.2e}", flush=True)
        ctx.close()
# round 2: the su(2) family (TMA midpoint, cp.async ring magnus, float32),
# the device analytic oracle, apply, the complex64 d = 2 register lanes,
# the Gauss-Legendre modes and the scaling-and-squaring extension
from cases import qubit_inputs  # noqa: E402
for prec, mode, pts in (("fp64", "midpoint", 5000), ("fp64", "magnus", 2001),
                        ("fp32", "midpoint", 3000), ("fp32", "simpson", 801)):
    h0, hs, v, dt = qubit_inputs(pts, mode)
    ctx = sp.create(prec)
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    u = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u
    print(f"su2 {prec} {mode}: {ctx.last_timing()['kernel']} det {abs(np.linalg.det(u)):.6f}",
          flush=True)
    ctx.close()
print("qubit reference", sp.midpoint_reference(sp.DrivenQubit(), 20000)[0, 0], flush=True)
rng = np.random.default_rng(1)
uu, _ = np.linalg.qr(rng.standard_normal((8, 8)) + 1j * rng.standard_normal((8, 8)))
psi = rng.standard_normal((5, 8)) + 1j * rng.standard_normal((5, 8))
print("apply", np.abs(sp.apply_batch(uu, psi) - psi @ uu.T).max(),
      np.abs(sp.apply(uu, np.outer(psi[0], psi[0].conj())) -
             uu @ np.outer(psi[0], psi[0].conj()) @ uu.conj().T).max(), flush=True)
h0, hs, v, dt = random_inputs(2, 2, 300, 3)
ctx = sp.create("fp32")
ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
print("f32 reg2", ctx.equiprop(sp.ControlAmplitudes(v, dt)).u[0, 0],
      ctx.last_timing()["kernel"], flush=True)
ctx.close()
for d in (8, 64):
    if NO_TMEM and d >= 64:
        continue
    h0, hs, v, dt = random_inputs(d, 2, 40 if d == 8 else 12, 5)
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=True, quadrature="gauss-legendre")
    print(f"gauss4 d={d}", ctx.equiprop(sp.ControlAmplitudes(v, dt / 2)).u[0, 0], flush=True)
    ctx.close()
h0, hs, v, dt = random_inputs(8, 2, 30, 6)
ctx = sp.create(scaling=True)
ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
res = ctx.equiprop(sp.ControlAmplitudes(v, 40 * dt))
print("scaling squarings", res.plan["squarings"], flush=True)
ctx.close()
# late round 2: multi-slice lanes (>= 3 slices per lane on the production
# grids) through the swizzled B / A layouts, the direct 256-bit publication
# and the release / acquire group barriers — the cross-slice reuse of the
# shared buffers and exchange buffers is what racecheck has to see
for d, n, algos in ((16, 3600, ("ps", "clenshaw")), (32, 900, ("ps", "clenshaw")),
                    (64, 444, ("ps3m", "ps")), (128, 111, ("ps3m",)), (256, 27, ("ps3m",))):
    for algo in algos:
        if NO_TMEM and algo == "ps3m":
            continue
        h0, hs, v, dt = random_inputs(d, 2, n, 11)
        ctx = sp.create()
        ctx.set_algorithm(algo)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        u = ctx.equiprop(sp.ControlAmplitudes(v, dt)).u
        print(f"multi-slice d={d} n={n} {algo}: {ctx.last_timing()['kernel']} lanes "
              f"{ctx.last_lanes()} unitarity {np.abs(u.conj().T @ u - np.eye(d)).max():.2e}",
              flush=True)
        ctx.close()
print("sanitize target done")
