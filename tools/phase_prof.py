"""Per-phase SM-clock breakdown of the group PS3 lane kernel (lane_ps3g_kernel).

    python tools/phase_prof.py [d] [n_ctrl] [slices]

Builds an instrumented copy of the library (-DSP_PHASE_PROF, clock64 stamps
by thread 0 of every CTA) into tools/libsliceprop_prof.so, runs one equiprop
and prints the share of CTA time in each phase of the slice loop.
"""
import ctypes
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "libsliceprop_prof.so")
spec = importlib.util.spec_from_file_location(
    "_sp_build", os.path.join(ROOT, "paper_2108_07126_b200", "build.py"))
bmod = importlib.util.module_from_spec(spec)
spec.loader.exec_module(bmod)
bmod.build(out=OUT, defines=("SP_PHASE_PROF",))
os.environ["SLICEPROP_B200_LIB"] = OUT
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2108_07126_b200 as sp  # noqa: E402
from cases import random_inputs  # noqa: E402

NAMES_PS = ["weights+assembly+sync", "T1 extract", "power GEMMs", "sync", "Clenshaw GEMMs",
            "U write+sync, tail", "P write+sync", "product GEMM", "power non-GEMM",
            "Clenshaw non-GEMM"]
NAMES = ["T1 extract", "power GEMMs", "publish 2y", "gsync1+frags", "Clenshaw GEMMs",
         "sync+publish U", "assemble next X+T1", "write P+gsync2", "product GEMM", "(unused)"]
d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 4
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
if d == 0:  # the driven qubit (C1)
    q = sp.DrivenQubit(1.0, 0.1, 1.0, 6.0)
    sysm = q.system()
    amp = q.amplitudes(n)
    h0, hs, v, dt = sysm.drift, list(sysm.controls), amp.values, amp.dt
else:
    h0, hs, v, dt = random_inputs(d, nc, n, 1)
ctx = sp.create()
ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
ctx.set_profiling(True)
amps = sp.ControlAmplitudes(v, dt)
ctx.equiprop(amps)
lib = sp._native.lib
buf = (ctypes.c_ulonglong * 16)()
tl = (ctypes.c_ulonglong * 4096)()
lib.sp_phase_prof(buf)
lib.sp_timeline(tl)
ctx.equiprop(amps)
lib.sp_phase_prof(buf)
lib.sp_timeline(tl)
t = ctx.last_timing()
tot = sum(buf[:10])
if not tot:
    sys.exit(f"d={d}: no phase data (kernel {ctx.last_timing()['kernel']} is not instrumented)")
print(f"d={d} N={nc} n={n}: kernel {t['main_kernel_ms']:.3f} ms ({t['kernel']})")
NAMES_SMALL = ["lane loop", "CTA tree", "publish+ticket", "tail (last CTA)"] + ["-"] * 6
names = NAMES if "ps3g" in t["kernel"] else NAMES_SMALL if "small" in t["kernel"] else NAMES_PS
for k, name in enumerate(names):
    print(f"  {name:18s} {100.0 * buf[k] / tot:6.2f} %  ({buf[k] / 1.965e3 / max(1, buf[15]):.2f} us per CTA of {buf[15]})")
ctx.close()

st = [tl[2 * i] for i in range(2048) if tl[2 * i]]
en = [tl[2 * i] + (tl[2 * i + 1] >> 8) for i in range(2048) if tl[2 * i]]
sm = [tl[2 * i + 1] & 0xff for i in range(2048) if tl[2 * i]]
if st:
    t0 = min(st)
    ss, ee = sorted(x - t0 for x in st), sorted(x - t0 for x in en)
    q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))] / 1e3
    print(f"  CTA timeline over {len(st)} CTAs (us from the first start): start p50 {q(ss, .5):.2f} "
          f"p90 {q(ss, .9):.2f} max {ss[-1] / 1e3:.2f}; end min {ee[0] / 1e3:.2f} p50 {q(ee, .5):.2f} "
          f"p90 {q(ee, .9):.2f} max {ee[-1] / 1e3:.2f}")
    if len(sys.argv) > 4:
        per = {}
        for x, e in zip(sm, en):
            per[x] = max(per.get(x, 0), e - t0)
        print("  last CTA end per SM (us): " + " ".join(f"{k}:{per[k] / 1e3:.1f}" for k in sorted(per)))
