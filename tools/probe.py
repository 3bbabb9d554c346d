"""Quick GPU probe: time the lane kernel per family (CUDA events inside the library)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np
import paper_2108_07126_b200 as sp
from cases import random_inputs, qubit_inputs

PEAK = 37.0e12
def run(label, h0, hs, v, dt, mode="midpoint", reps=3, algo="auto"):
    ctx = sp.create(); ctx.set_algorithm(algo); ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                                           quadrature=None if mode == "magnus" else mode)
    ctx.set_profiling(True)
    amps = sp.ControlAmplitudes(v, dt)
    r = ctx.equiprop(amps)
    best = 1e9; wall = 1e9
    for _ in range(reps):
        t0 = time.perf_counter(); ctx.equiprop(amps); wall = min(wall, time.perf_counter() - t0)
        t = ctx.last_timing(); best = min(best, t["main_kernel_ms"])
    n = r.slice_count; m = r.plan["m_max"]; d = h0.shape[0]
    canon = n * (8 * d**3 * (m + 1) + 4 * d * d * (len(hs) + 1))
    print(f"{label}: n={n} m={m} kernel {best:.3f} ms ({t['kernel']}), wall {wall*1e3:.2f} ms, "
          f"slices/s {n/(best/1e3):.3e}, canon TF {canon/(best/1e3)/1e12:.2f} ({canon/(best/1e3)/PEAK*100:.1f}%), "
          f"exec TF {t['executed_flops']/(best/1e3)/1e12:.2f}, launches {t['launches']}", flush=True)
    ctx.close()

run("d2 qubit 1e5", *qubit_inputs(100000, "midpoint"))
run("d2 qubit 1e6", *qubit_inputs(1000000, "midpoint"))
run("d2 rand 1e6", *random_inputs(2, 2, 1000000, 1))
run("d4 rand 1e6", *random_inputs(4, 2, 1000000, 1))
run("d16 rand 1e5", *random_inputs(16, 2, 100000, 1))
run("d32 rand 1e5", *random_inputs(32, 2, 100000, 1))
run("d64 rand 2e4", *random_inputs(64, 2, 20000, 1))
run("d128 rand 4e3", *random_inputs(128, 4, 4000, 1))
run("d256 rand 500", *random_inputs(256, 4, 500, 1))
if len(sys.argv) > 1 and sys.argv[1] == "algos":
    for a in ("ps", "ps3m"):
        run(f"d32 rand 1e5 {a}", *random_inputs(32, 2, 100000, 1), algo=a)
        run(f"d64 rand 2e4 {a}", *random_inputs(64, 2, 20000, 1), algo=a)
        run(f"d128 rand 4e3 {a}", *random_inputs(128, 4, 4000, 1), algo=a)
if len(sys.argv) > 1 and sys.argv[1] == "big":
    run("d512 rand 64", *random_inputs(512, 4, 64, 1), reps=2)
    run("d384 rand 64", *random_inputs(384, 4, 64, 1), reps=2)
if len(sys.argv) > 1 and sys.argv[1] == "cum":
    for d, n_ctrl, n in ((2, 2, 1000000), (4, 2, 200000), (16, 2, 100000), (32, 2, 50000),
                         (64, 2, 10000), (128, 4, 2000)):
        h0, hs, v, dt = random_inputs(d, n_ctrl, n, 1)
        ctx = sp.create(); ctx.set_hamiltonian(sp.ControlSystem(h0, hs)); ctx.set_profiling(True)
        amps = sp.ControlAmplitudes(v, dt)
        ctx.equiprop_all(amps)
        t0 = time.perf_counter(); cum = ctx.equiprop_all(amps); wall = time.perf_counter() - t0
        lane_ms = ctx.last_timing()["main_kernel_ms"]
        seq = ctx.equiprop(amps, reduction="sequential").u
        out_gb = cum.u_all.nbytes / 1e9
        print(f"cum d{d} n={n}: wall {wall*1e3:.2f} ms (lane kernel {lane_ms:.2f} ms), output "
              f"{out_gb:.3f} GB, final==seq {np.array_equal(cum.final, seq)}", flush=True)
        ctx.close()
if len(sys.argv) > 1 and sys.argv[1] == "d8":
    for d in (5, 8):
        for a in ("auto", "clenshaw", "ps", "ps3m"):
            run(f"d{d} rand 1e6 {a}", *random_inputs(d, 2, 1000000, 1), algo=a)
if len(sys.argv) > 1 and sys.argv[1] == "magnus":
    run("d128 magnus 2e3", *random_inputs(128, 4, 4001, 1), mode="magnus")
    run("d32 magnus 2e4", *random_inputs(32, 2, 40001, 1), mode="magnus")
if len(sys.argv) > 1 and sys.argv[1] == "c64":
    for d, n in ((16, 100000), (32, 100000), (12, 100000), (24, 50000)):
        h0, hs, v, dt = random_inputs(d, 2, n, 1)
        for prec in ("fp32", "fp64"):
            ctx = sp.create(prec); ctx.set_hamiltonian(sp.ControlSystem(h0, hs)); ctx.set_profiling(True)
            amps = sp.ControlAmplitudes(v, dt)
            u = ctx.equiprop(amps).u
            best = 1e9
            for _ in range(3):
                ctx.equiprop(amps); best = min(best, ctx.last_timing()["main_kernel_ms"])
            t = ctx.last_timing()
            print(f"c64 probe d{d} {prec}: n={n} kernel {best:.3f} ms ({t['kernel']}), slices/s {n/(best/1e3):.3e}", flush=True)
            ctx.close()
