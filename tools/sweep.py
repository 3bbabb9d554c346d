"""C5 sweep (BASELINE.json configs[4]): dim 2..512 x slices 1e3..1e7, complex64
and complex128, one B200, with the CPU reference algorithm timed beside it.

    python tools/sweep.py [--out gpurun_out/sweep.jsonl] [--cap-s 6] [--cpu-s 2]

Each GPU point is the device-resident path (``equiprop_device_ptr``: the
amplitude table already in HBM, CUDA events on the launching stream, median
of up to 3 steps after one warm-up).  Systems are the random unit-1-norm
drift + 2 controls of C3(i) (seed 20240911, beta = 0.5 -> m = 13 fp64 / 7
fp32), midpoint.  Points whose estimated GPU time exceeds --cap-s are skipped
(d = 512 x 1e6 would take ~10 min).  The CPU column is the reference
itself (sliceprop from baseline/_ref through its public API, numpy/OpenBLAS
on all host threads; bench.CpuArm, the oracle port only if the install is
missing) on a bounded prefix of the same system, one rate per (dim,
precision): its runtime is linear in the slice count (reference property,
test_acceptance.py:229-245).  ``frac`` = executed flops of the lane kernel /
its duration / the measured peak of the pipe it runs on (FP64 DMMA for the
tensor-core families, FP64 DFMA for the d <= 4 register families, FP32 FFMA
for the complex64 d <= 8 kernel); ``canonical_frac`` = the reference-algorithm
work F(d, m, T) on the same denominator.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

DIMS = [2, 4, 8, 16, 32, 64, 128, 256, 512]
SLICES = [1_000, 10_000, 100_000, 1_000_000, 10_000_000]
N_CTRL = 2
SEED = 20240911


def canonical_flops(d, m, n_terms):
    return 8.0 * d ** 3 * (m + 1) + 4.0 * d * d * n_terms


def cpu_rate(h0, hs, values, dt, bits, target_s):
    """(slices/s, prefix slices, kind) of the reference on the host cores."""
    import bench
    arm = bench.CpuArm(h0, hs, dt, "midpoint")
    if bits == 32:
        if arm.ref is not None:
            arm.ctx.close()
            arm.ctx = arm.ref.create(precision="fp32")
            arm.ctx.set_hamiltonian(arm.ref.ControlSystem(h0, hs))
        else:
            import oracle
            arm.run = lambda v, reduction="pairwise": oracle.equiprop(
                h0, hs, v, dt, bits=32, reduction=reduction)[0]
    s = arm.sample(values[:min(values.shape[0], 2_000_000)], target_s, repeats=1)
    arm.close()
    return s["rate"], s["slices"], arm.kind


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.jsonl"))
    ap.add_argument("--cap-s", type=float, default=6.0)
    ap.add_argument("--cpu-s", type=float, default=2.0)
    ap.add_argument("--dims", default=",".join(map(str, DIMS)))
    ap.add_argument("--precisions", default="fp64,fp32")
    ap.add_argument("--qubit", type=int, default=1, help="add the driven-qubit d = 2 series")
    ap.add_argument("--modes", default="midpoint,simpson,magnus",
                    help="slicing modes (three-point modes: fp64 rows)")
    args = ap.parse_args()
    import torch

    import paper_2108_07126_b200 as sp
    from cases import unit_hermitian

    with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
        peaks = json.load(fh)

    def pipe_peak(kernel):
        key = ("fp32_ffma_tflops" if kernel.startswith(("lane_f32", "lane_su2_f32"))
               else "fp64_dfma_tflops" if kernel.startswith(("lane_small", "lane_su2"))
               else "fp64_dmma_tflops")
        return peaks[key] * 1e12
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    fh = open(args.out, "w")
    nmax = max(SLICES)
    combos = [(p, "midpoint") for p in args.precisions.split(",")]
    combos += [("fp64", m) for m in args.modes.split(",") if m and m != "midpoint"]
    for prec, mode in combos:
        bits = 64 if prec == "fp64" else 32
        three = mode != "midpoint"
        for d in map(int, args.dims.split(",")):
            rng = np.random.default_rng(SEED)
            h0 = unit_hermitian(rng, d)
            hs = [unit_hermitian(rng, d) for _ in range(N_CTRL)]
            dt = 0.5 / (N_CTRL + 1.0) / (2.0 if three else 1.0)
            values = rng.uniform(-1.0, 1.0, ((2 * nmax + 1) if three else nmax, N_CTRL))
            ctx = sp.create(prec)
            ctx.set_hamiltonian(sp.ControlSystem(h0, hs), magnus=mode == "magnus",
                                quadrature=None if mode == "magnus" else mode)
            ctx.set_profiling(True)
            plan = ctx.plan_for(dt)
            n_terms = 1 + 2 * N_CTRL + N_CTRL * (N_CTRL - 1) // 2 if mode == "magnus" \
                else N_CTRL + 1
            F = canonical_flops(d, plan.m_max, n_terms)
            d_amps = torch.from_numpy(values).to(dev)
            out = torch.empty((d, d), dtype=torch.complex128 if bits == 64 else torch.complex64,
                              device=dev)
            rate_est = None
            if three:  # the CPU column is the midpoint reference's
                cpu, cpu_n, cpu_kind = None, 0, "n/a (three-point row)"
            else:
                cpu, cpu_n, cpu_kind = cpu_rate(h0, hs, values, dt, bits, args.cpu_s)
            for n in SLICES:
                if rate_est is not None and n / rate_est > args.cap_s:
                    rec = {"precision": prec, "dim": d, "slices": n, "mode": mode, "skipped":
                           f"estimated {n / rate_est:.0f} s > cap {args.cap_s} s"}
                    print(json.dumps(rec), flush=True)
                    fh.write(json.dumps(rec) + "\n")
                    continue

                pts = 2 * n + 1 if three else n

                def step():
                    ctx.equiprop_device_ptr(d_amps.data_ptr(), pts, N_CTRL, dt, out.data_ptr(),
                                            stream=stream.cuda_stream, plan=plan)
                step()
                torch.cuda.synchronize(dev)
                ms, kern = [], []
                for _ in range(3):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    step()
                    e1.record(stream)
                    torch.cuda.synchronize(dev)
                    ms.append(e0.elapsed_time(e1))
                    t = ctx.last_timing()
                    kern.append(t["main_kernel_ms"])
                    if ms[-1] > 1500:
                        break
                step_ms = statistics.median(ms)
                rate = n / (step_ms / 1e3)
                rate_est = rate
                kms = statistics.median(kern)
                rec = {"precision": prec, "dim": d, "slices": n, "mode": mode, "m": plan.m_max,
                       "slices_per_s": rate, "ms_per_step": step_ms,
                       "kernel": t["kernel"], "kernel_ms": kms, "launches": t["launches"],
                       "canonical_tflops": n * F / (step_ms / 1e3) / 1e12,
                       "frac": t["executed_flops"] / (kms / 1e3) / pipe_peak(t["kernel"]),
                       "canonical_frac": n * F / (kms / 1e3) / pipe_peak(t["kernel"]),
                       "series": ctx.last_algorithm(), "lanes": ctx.last_lanes(),
                       "cpu_slices_per_s": cpu, "cpu_sample_slices": cpu_n,
                       "cpu_kind": cpu_kind,
                       "gpu_over_cpu": rate / cpu if cpu else None}
                print(json.dumps(rec), flush=True)
                fh.write(json.dumps(rec) + "\n")
                fh.flush()
            ctx.close()
            del d_amps
        if args.qubit and mode == "midpoint":
            qubit_series(args, prec, sp, torch, dev, stream, fh, pipe_peak)
    fh.close()


def qubit_series(args, prec, sp, torch, dev, stream, fh, pipe_peak):
    """The paper's driven qubit (d = 2, su(2) terms: the quaternion kernel for
    fp64) at every slice count: the north-star d = 2 series.  Each point is
    timed like the bench's qubit lines (CUDA graph, L2 written then read
    between 30 replays, mean over the replays); ``hbm_frac`` = amplitude
    bytes / kernel-bounded step time / the measured copy bandwidth."""
    from cases import qubit_inputs
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = float(json.load(f)["hbm_gbs"]) * 1e9
    except (OSError, ValueError, KeyError):
        hbm = 6.65e12
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    st = torch.cuda.Stream(dev)
    for n in SLICES:
        h0, hs, values, dt = qubit_inputs(n, "midpoint")
        ctx = sp.create(prec)
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        plan = ctx.plan_for(dt)
        d_amps = torch.from_numpy(values).to(dev)
        out = torch.empty((2, 2), dtype=torch.complex128 if prec == "fp64" else torch.complex64,
                          device=dev)
        with torch.cuda.stream(st):
            for _ in range(3):
                ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                        stream=st.cuda_stream, plan=plan)
        torch.cuda.synchronize(dev)
        ctx.set_profiling(True)
        ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                stream=st.cuda_stream, plan=plan)
        torch.cuda.synchronize(dev)
        t = ctx.last_timing()
        ctx.set_profiling(False)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            ctx.equiprop_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                    stream=st.cuda_stream, plan=plan)
        ts = []
        with torch.cuda.stream(st):
            for k in range(33):
                flush.fill_(float(k))
                clean.sum()
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(st)
                g.replay()
                b.record(st)
                st.synchronize()
                if k >= 3:
                    ts.append(a.elapsed_time(b))
        step_ms = statistics.mean(ts)
        F = canonical_flops(2, plan.m_max, 3)
        rec = {"precision": prec, "dim": 2, "system": "driven qubit", "slices": n,
               "m": plan.m_max, "slices_per_s": n / (step_ms / 1e3), "ms_per_step": step_ms,
               "kernel": t["kernel"], "fp64_frac": t["executed_flops"] / (step_ms / 1e3)
               / pipe_peak(t["kernel"]),
               "canonical_frac": n * F / (step_ms / 1e3) / pipe_peak(t["kernel"]),
               "hbm_frac": n * 16 / (step_ms / 1e3) / hbm,
               "timing": "CUDA graph, L2 flushed, mean of 30 replays (step, not kernel)"}
        print(json.dumps(rec), flush=True)
        fh.write(json.dumps(rec) + "\n")
        fh.flush()
        ctx.close()


if __name__ == "__main__":
    main()
