#!/usr/bin/env python
"""Benchmark of the equiprop hot path on B200 (contract: see DESIGN.md §7).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)

Headline workload (BASELINE.json configs[3], the largest single-GPU config):
C4 = dim-128 random unit-1-norm system, 4 controls, 1e6 slices, midpoint,
complex128, beta = 0.5 (m = 13), time-sharded over the N GPUs (strong
scaling: 1e6 slices in total).  Secondary lines (same JSON, "per_dim"): the
C4 magnus variant (pts = 2e6 + 1, 15 expansion terms, m = 15), C3 (dim 32,
2 controls, 1e6 slices; random and the coupled-spin chain of configs[2]), C1
(the paper's driven qubit, dim 2, 1e5 slices) and c1m (the same qubit at the
north star's 1e6 slices).  A step is one full propagation U = U_{n-1} ... U_0
of the workload; value = slices / device time (CUDA events, max over ranks),
with the amplitude table resident in HBM and L2 flushed between timed steps.
e2e = the same through the public API with the table in page-locked host
memory (H2D + kernels + gather + D2H inside the timed region, wall clock,
max over ranks).

The CPU side is the UNMODIFIED reference (sliceprop 0.1.0, pure Python +
numpy/OpenBLAS) installed under baseline/_ref (tools/install_reference.sh),
driven through its own public API (create / set_hamiltonian / equiprop) on a
bounded prefix of the same workload; the oracle port (oracle/) stands in only
if that install is missing.  The same prefix run on the GPU gives the
``parity`` object of every line (rel-Frobenius vs the reference, with the
reference's own pairwise-vs-sequential noise eps_self beside it).
``--impl reference`` is that CPU arm alone; it never imports this package.
"""

from __future__ import annotations

import argparse
import contextlib
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
REF_DIR = os.path.join(ROOT, "baseline", "_ref")

METRIC = "time slices/sec (complex128) at dim 2/32/128, 1/2/4/8 B200; % FP64 roofline"
UNIT = "slices/s"
SEED = 20240911

WORKLOADS = {
    "c4": dict(d=128, n_ctrl=4, slices=1_000_000, kind="random", mode="midpoint",
               label="C4: dim-128 random unit-norm system, 4 controls, 1e6 slices, midpoint, "
                     "complex128, beta=0.5 (m=13)"),
    "c4m": dict(d=128, n_ctrl=4, slices=1_000_000, kind="random", mode="magnus",
                label="C4 magnus variant: dim-128 random unit-norm system, 4 controls, "
                      "pts=2e6+1 (1e6 doubled steps), 4th-order Magnus (15 terms), "
                      "complex128 (m=15)"),
    "c3": dict(d=32, n_ctrl=2, slices=1_000_000, kind="random", mode="midpoint",
               label="C3: dim-32 random unit-norm system, 2 controls, 1e6 slices, midpoint, "
                     "complex128, beta=0.5 (m=13)"),
    "c3s": dict(d=32, n_ctrl=2, slices=1_000_000, kind="spin", mode="midpoint",
                label="C3 physics variant: 5-spin coupled chain (d=32, 2 controls, "
                      "cos/sin drive over T=6), 1e6 slices, midpoint, complex128"),
    "c1": dict(d=2, n_ctrl=2, slices=100_000, kind="qubit", mode="midpoint",
               label="C1: paper's driven qubit (w0=1, w1=0.1, wrf=1, T=6), dim 2, 2 controls, "
                     "1e5 slices, midpoint, complex128 (m=3)"),
    "c1m": dict(d=2, n_ctrl=2, slices=1_000_000, kind="qubit", mode="midpoint",
                label="north-star d=2 target: the driven qubit at 1e6 slices, midpoint, "
                      "complex128 (m=3)"),
}

# secondary lines whose steps are seconds long run fewer timed steps; the
# microsecond-scale ones more (CUDA event timestamps tick in ~2 us steps on
# this B200, so a mean over many steps is needed)
SECONDARY_MAX_STEPS = {"c4m": 5}
SECONDARY_MIN_STEPS = {"c1": 50, "c1m": 50, "c3": 10, "c3s": 10}


def fp64_peaks():
    with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
        return json.load(fh)


# ---------------------------------------------------------------------------
# synthetic inputs (numpy only: the reference arm must not load this package)
# ---------------------------------------------------------------------------

PAULI_X = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)
PAULI_Y = np.array([[0.0, -1.0j], [1.0j, 0.0]], dtype=complex)
PAULI_Z = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=complex)


def _one_norm(m):
    return float(np.abs(m).sum(axis=0).max())


def _site_op(p, i, n):
    out = np.ones((1, 1), dtype=complex)
    for k in range(n):
        out = np.kron(out, p if k == i else np.eye(2, dtype=complex))
    return out


def _drive(pts, mode, duration=6.0, wrf=1.0):
    """DrivenQubit sampling (reference studies.py:77-90)."""
    if mode == "midpoint":
        dt = duration / max(pts, 1)
        t = (np.arange(pts) + 0.5) * dt
    else:
        dt = duration / (pts - 1)
        t = np.arange(pts) * dt
    return np.column_stack([np.cos(wrf * t), np.sin(wrf * t)]), dt


def make_problem(wl):
    """(H0, [H_k], amplitude table, dt) — deterministic synthetic inputs.

    random: reference bench_grid's unit 1-norm systems (studies.py:248-253)
    with N controls, seed 20240911, dt = 0.5 / sum of 1-norms (beta = 0.5 for
    midpoint), uniform(-1, 1) amplitudes; qubit: DrivenQubit(1, 0.1, 1, 6)
    (studies.py:51-90); spin: the 5-spin chain of SpinChain."""
    mode = wl["mode"]
    pts = wl["slices"] if mode == "midpoint" else 2 * wl["slices"] + 1
    if wl["kind"] == "qubit":
        values, dt = _drive(pts, mode)
        return (0.5 * PAULI_Z, [0.05 * PAULI_X, 0.05 * PAULI_Y],
                np.ascontiguousarray(values), dt)
    if wl["kind"] == "spin":
        n = 5
        h0 = sum(0.5 * (1.0 + 0.05 * i) * _site_op(PAULI_Z, i, n) for i in range(n))
        for i in range(n - 1):
            for p in (PAULI_X, PAULI_Y, PAULI_Z):
                h0 = h0 + 0.025 * (_site_op(p, i, n) @ _site_op(p, i + 1, n))
        hx = sum(0.05 * _site_op(PAULI_X, i, n) for i in range(n))
        hy = sum(0.05 * _site_op(PAULI_Y, i, n) for i in range(n))
        values, dt = _drive(pts, mode)
        return h0, [hx, hy], np.ascontiguousarray(values), dt
    rng = np.random.default_rng(SEED)
    d = wl["d"]

    def unit_hermitian():
        a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
        h = 0.5 * (a + a.conj().T)
        return h / _one_norm(h)

    h0 = unit_hermitian()
    hs = [unit_hermitian() for _ in range(wl["n_ctrl"])]
    dt = 0.5 / sum(_one_norm(h) for h in [h0, *hs])
    values = rng.uniform(-1.0, 1.0, (pts, wl["n_ctrl"]))
    return h0, hs, values, dt


def canonical_flops(d, m, n_terms):
    """F(d, m, T) = 8 d^3 (m + 1) + 4 d^2 T per slice."""
    return 8.0 * d ** 3 * (m + 1) + 4.0 * d * d * n_terms


def n_terms_for(wl):
    n = wl["n_ctrl"]
    return 2 * n + n * (n - 1) // 2 + 1 if wl["mode"] == "magnus" else n + 1


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], 0.0, set()
        for line in (getattr(self, "out", "") or "").splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# the CPU side: the unmodified reference (baseline/_ref), else the oracle port
# ---------------------------------------------------------------------------

def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()
                    if i.get("user_api") == "blas"), default=1)
    except Exception:
        return os.cpu_count() or 1


class CpuArm:
    """One equiprop of the reference on a prefix of the workload.

    kind "reference": ``sliceprop`` imported from baseline/_ref through its
    public API (create / set_hamiltonian / ControlAmplitudes / equiprop,
    propagator.py:279-308); kind "port": the oracle restatement."""

    def __init__(self, h0, hs, dt, mode):
        self.h0, self.hs, self.dt, self.mode = h0, hs, dt, mode
        self.kind, self.ref, self.where = "port", None, "oracle/ (numpy restatement)"
        if os.path.isdir(os.path.join(REF_DIR, "sliceprop")):
            if REF_DIR not in sys.path:
                sys.path.insert(0, REF_DIR)
            try:
                import sliceprop
                if os.path.abspath(sliceprop.__file__).startswith(REF_DIR):
                    self.ref, self.kind = sliceprop, "reference"
                    self.where = f"sliceprop {getattr(sliceprop, '__version__', '?')} " \
                                 "(baseline/_ref, unmodified reference)"
            except Exception as exc:  # fall back to the port, say why
                self.where = f"oracle/ (reference import failed: {exc})"
        if self.ref is not None:
            self.ctx = self.ref.create()
            self.ctx.set_hamiltonian(self.ref.ControlSystem(h0, hs), magnus=mode == "magnus",
                                     quadrature=None if mode == "magnus" else mode)

    def pts_for(self, slices):
        return slices if self.mode == "midpoint" else 2 * slices + 1

    def run(self, values, reduction="pairwise"):
        if self.ref is not None:
            amps = self.ref.ControlAmplitudes(values, self.dt)
            return self.ctx.equiprop(amps, reduction=reduction).u
        import oracle
        u, _, _ = oracle.equiprop(self.h0, self.hs, values, self.dt, mode=self.mode,
                                  reduction=reduction)
        return u

    def sample(self, values, target_s, repeats=3, max_slices=2_000_000):
        """Bounded sample: one calibration call, then `repeats` timed calls of
        the prefix sized to ~target_s / repeats each.  Returns a dict with the
        rate, the prefix length and its pairwise output."""
        n_avail = values.shape[0] if self.mode == "midpoint" else (values.shape[0] - 1) // 2
        n0 = min(n_avail, 64 if self.h0.shape[0] >= 64 else 2048)
        t0 = time.perf_counter()
        self.run(values[:self.pts_for(n0)])
        per = (time.perf_counter() - t0) / n0
        n = int(max(n0, min(max_slices, n_avail, target_s / repeats / max(per, 1e-9))))
        prefix = values[:self.pts_for(n)]
        times, u = [], None
        for _ in range(repeats):
            t0 = time.perf_counter()
            u = self.run(prefix)
            times.append(time.perf_counter() - t0)
        sec = statistics.median(times)
        return {"rate": n / sec, "slices": n, "sec": sec, "repeats": repeats, "u": u,
                "prefix": prefix, "threads": blas_threads()}

    def baseline(self, s, full_slices):
        return {"value": s["rate"], "unit": UNIT, "cores": s["threads"], "kind": self.kind,
                "sample": f"first {s['slices']} of {full_slices} slices of the workload "
                          f"({'full workload' if s['slices'] >= full_slices else 'prefix'}), "
                          f"median of {s['repeats']} calls ({s['sec']:.2f} s each) of "
                          f"{self.where}, OpenBLAS {s['threads']} threads on "
                          f"{os.cpu_count()} host cpus"}

    def close(self):
        if self.ref is not None:
            self.ctx.close()


def run_reference(args):
    """--impl reference: rank 0 times the reference on the host cores (the
    other ranks exit without work).  Never imports paper_2108_07126_b200."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    wl = WORKLOADS[args.workload]
    h0, hs, values, dt = make_problem(wl)
    arm = CpuArm(h0, hs, dt, wl["mode"])
    cal = arm.sample(values, args.cpu_seconds, repeats=1)
    n = cal["slices"]
    prefix = cal["prefix"]
    for _ in range(args.warmup):
        arm.run(prefix[:arm.pts_for(max(1, n // 4))])
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        arm.run(prefix)
        times.append(time.perf_counter() - t0)
    rate = n / statistics.median(times)
    threads = blas_threads()
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wl["slices"] / rate * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
        "config": {"workload": wl["label"], "dim": wl["d"], "n_ctrl": wl["n_ctrl"],
                   "slices": wl["slices"], "mode": wl["mode"],
                   "sample_slices_per_step": n, "same_config": n >= wl["slices"],
                   "note": "each step propagates the first sample_slices_per_step slices; "
                           "ms_per_step is extrapolated linearly to the full workload "
                           "(linear runtime: reference test_acceptance.py:229-245)"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": arm.kind,
                         "sample": f"first {n} slices of the workload per step, median of "
                                   f"{args.steps} steps, {arm.where}, OpenBLAS {threads} "
                                   f"threads, host {os.cpu_count()} cpus"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    arm.close()
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# the B200 arm
# ---------------------------------------------------------------------------

def max_over_ranks(dist, vals, dev):
    import torch
    on = dev if dist.get_backend() == "nccl" else "cpu"
    red = torch.tensor(vals, dtype=torch.float64, device=on)
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    return red.tolist()


def roofline_for(t, local_slices, wl, m, kern_ms, peaks):
    """Dominant-kernel roofline.  frac = EXECUTED FP64 flops of the launch
    (the instructions the kernel issues: PS / 3M forms, Cayley-Hamilton
    pairs) / duration / the measured peak of the pipe it runs on (DFMA for
    the register families d <= 4, DMMA above); canonical_frac = the
    reference-algorithm work F(d, m, T) of SURVEY.md §8(d) on the same
    denominator (above 1 when the kernel needs fewer flops than the
    reference's Clenshaw count)."""
    ffma = t["kernel"].startswith(("lane_f32", "lane_su2_f32"))
    dfma = not ffma and t["kernel"].startswith(("lane_small", "lane_su2"))
    peak = (peaks["fp32_ffma_tflops"] if ffma else peaks["fp64_dfma_tflops"] if dfma
            else peaks["fp64_dmma_tflops"]) * 1e12
    F = canonical_flops(wl["d"], m, n_terms_for(wl))
    executed = t["executed_flops"] / (kern_ms / 1e3)
    canonical = local_slices * F / (kern_ms / 1e3)
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            cap = json.load(fh).get(t["kernel"])
        if cap:
            traffic = cap["dram_bytes"] * local_slices / cap["slices"]
            how = ("measured on one launch of this size" if cap["slices"] == local_slices else
                   f"measured at {cap['slices']} slices, scaled linearly to this launch")
            traffic_note = (f"ncu dram__bytes_read.sum + dram__bytes_write.sum "
                            f"({cap['dram_bytes']:.4g} B; {cap.get('source', '')}), {how}; "
                            f"algorithmic bytes/slice = {8 * wl['n_ctrl']} (amplitude row)")
    except (OSError, ValueError, KeyError):
        pass
    # amplitude bytes of the launch (midpoint: one row per slice; three-point
    # modes: two new rows per slice) against the measured HBM copy bandwidth
    rows = local_slices * (1 if wl["mode"] == "midpoint" else 2)
    amp_bytes = rows * 8 * wl["n_ctrl"]
    hbm_gbs = amp_bytes / (kern_ms / 1e3) / 1e9
    hbm_peak = measured_hbm_gbs()
    line = {"bound": "tensor", "achieved": executed / 1e12, "peak": peak / 1e12,
            "unit": "TFLOP/s", "frac": executed / peak, "traffic": traffic,
            "traffic_note": traffic_note, "kernel": t["kernel"], "kernel_ms": kern_ms,
            "executed_flops_per_launch": t["executed_flops"],
            "canonical_achieved": canonical / 1e12, "canonical_frac": canonical / peak,
            "canonical_flops_per_launch": local_slices * F,
            "pipe": "FP32 FFMA (CUDA cores)" if ffma else "FP64 DFMA (CUDA cores)" if dfma
                    else "FP64 DMMA (mma.sync f64)",
            "peak_source": "measured " + ("FP32 FFMA" if ffma else "FP64 DFMA" if dfma
                                          else "FP64 DMMA")
                           + " peak (tools/fp64_peak.cu, profiles/fp64_peak.json; "
                             "MEASURED_PEAKS.json has no FP64 entry)",
            "amplitude_bytes_per_launch": amp_bytes, "hbm_achieved_gbs": hbm_gbs,
            "hbm_peak_gbs": hbm_peak, "hbm_frac": hbm_gbs / hbm_peak if hbm_peak else None,
            "pipe_frac": executed / peak}
    if hbm_peak and hbm_gbs / hbm_peak > executed / peak:
        # the su(2) quaternion kernel executes ~34 FP64 instructions per 16-byte
        # amplitude row: its bound is the amplitude stream, not the FP64 pipe
        line.update({"bound": "hbm", "achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": hbm_gbs / hbm_peak,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (driver-measured copy "
                                    "bandwidth)"})
    return line


def measured_hbm_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0  # B200_PROFILING.md fallback ("of fallback")


def measure_gpu(args, name, rank, world, local_rank, dist, headline):
    import torch

    import paper_2108_07126_b200 as sp
    from paper_2108_07126_b200.sharding import (equiprop_sharded_device, partition,
                                                shard_rows)
    wl = WORKLOADS[name]
    steps = args.steps if headline else max(min(args.steps, SECONDARY_MAX_STEPS.get(name, 10**9)),
                                            SECONDARY_MIN_STEPS.get(name, 0))
    h0, hs, values, dt = make_problem(wl)
    mode = wl["mode"]
    system = sp.ControlSystem(h0, hs)
    d = system.dim
    n = wl["slices"]
    ctx = sp.create(device=local_rank)
    ctx.set_hamiltonian(system, magnus=mode == "magnus",
                        quadrature=None if mode == "magnus" else mode)
    ctx.set_profiling(True)
    plan = ctx.plan_for(dt)
    a, b = partition(n, world)[rank]
    lo, hi = shard_rows(mode, a, b)
    local = np.ascontiguousarray(values[lo:hi])
    dev = torch.device("cuda", local_rank)
    d_amps = torch.from_numpy(local.copy()).to(dev)
    out = torch.empty((d, d), dtype=torch.complex128, device=dev)
    # L2 flush between timed steps: write 256 MiB (> 126 MB L2), then read
    # another 256 MiB so the write-backs of the flush itself finish before
    # the timed region (L2 left cold for the inputs and clean)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    clean = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device=dev)

    def l2_flush(k):
        flush.fill_(float(k))
        clean.sum()
    # one non-default stream for the step, the flush and the events (the
    # legacy default stream adds ~2 us of implicit synchronisation per step)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    # amplitude validation (|c| <= 1) is part of the job: it runs inside the
    # lane kernel and its flag is read after each timed step
    def validate():
        if ctx.amplitude_violation() >= 0:
            raise sp.AmplitudeBoundError("amplitude outside [-1, 1]")

    def step():
        if world == 1:
            ctx.equiprop_device_ptr(d_amps.data_ptr(), hi - lo, wl["n_ctrl"], dt,
                                    out.data_ptr(), stream=stream.cuda_stream, plan=plan)
            return out
        res, _, _ = equiprop_sharded_device(ctx, d_amps, dt, n, stream=stream)
        return res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    t = ctx.last_timing()
    launches_per_step = t["launches"]
    lanes = ctx.last_lanes()
    # launch-latency-bound secondary workloads (C1: ~10 us of GPU work per
    # step) replay the step as a CUDA graph, the way a serving loop would;
    # the headline step (seconds of GPU work) is launched directly
    graph = None
    if world == 1 and not headline and not args.no_graph and wl["d"] <= 32:
        try:
            ctx.set_profiling(False)
            torch.cuda.synchronize(dev)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                ctx.equiprop_device_ptr(d_amps.data_ptr(), hi - lo, wl["n_ctrl"], dt,
                                        out.data_ptr(), stream=stream.cuda_stream, plan=plan)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as exc:  # capture not possible: time direct launches
            print(f"[bench] CUDA graph capture failed ({exc}); direct launches",
                  file=sys.stderr)
            graph = None
            ctx.set_profiling(True)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(steps)]
    kernel_ms, launches = [], 0
    # clocks are sampled (nvidia-smi every 200 ms) during the headline's
    # timed region; the microsecond secondaries run without the poller
    clk = Clocks(local_rank) if headline else None
    with (clk if clk is not None else contextlib.nullcontext()):
        for k in range(steps):
            l2_flush(k)
            evs[k][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            evs[k][1].record(stream)
            stream.synchronize()
            if graph is not None:
                launches += launches_per_step
            else:
                tk = ctx.last_timing()
                kernel_ms.append(tk["main_kernel_ms"])
                launches += tk["launches"]
            # the in-kernel amplitude check's flag (a blocking D2H read) is
            # fetched after every step for the headline; the microsecond
            # secondaries read it once after the timed loop (same table
            # every step, so the flag is the same)
            if headline:
                validate()
        torch.cuda.synchronize(dev)
        validate()
    if graph is not None:  # kernel time bounded by the replayed step
        kernel_ms = [s.elapsed_time(e) for s, e in evs]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    step_ms = [s.elapsed_time(e) for s, e in evs]
    total_ms = sum(step_ms)
    kern = statistics.mean(kernel_ms)
    if dist is not None:
        total_ms, kern = max_over_ranks(dist, [total_ms, kern], dev)
    value = n * steps / (total_ms / 1e3)
    roofline = roofline_for(t, b - a, wl, plan.m_max, kern, fp64_peaks())

    # ---- e2e: public API, page-locked host table, H2D + compute + D2H timed
    pinned = torch.empty(local.shape, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = local
    e2e_times = []
    amps_obj = sp.ControlAmplitudes(pinned.numpy(), dt, copy=False) if world == 1 else None
    u = None
    for k in range(args.warmup + steps):
        l2_flush(k)
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        if world == 1:
            u = ctx.equiprop(amps_obj).u
        else:
            d_loc = pinned.to(dev, non_blocking=True)
            res, _, _ = equiprop_sharded_device(ctx, d_loc, dt, n, stream=stream)
            u = res.cpu().numpy()
        t1 = time.perf_counter()
        if k >= args.warmup:
            e2e_times.append(t1 - t0)
    e2e_s = sum(e2e_times)
    if dist is not None:
        (e2e_s,) = max_over_ranks(dist, [e2e_s], dev)
    e2e = {"value": n * steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(local.nbytes), "d2h_bytes_per_step": int(d * d * 16),
           "ms_per_step": e2e_s / steps * 1e3}
    assert np.all(np.isfinite(u))
    res = {"value": value, "ms_per_step": total_ms / steps, "steps": steps,
           "roofline": roofline, "e2e": e2e, "gpu_launches": launches,
           "clocks": clk.summary() if clk is not None else None, "m": plan.m_max, "lanes": lanes,
           "config": {"workload": wl["label"], "dim": d, "n_ctrl": wl["n_ctrl"],
                      "slices": n, "mode": mode, "m": plan.m_max,
                      "n_terms": n_terms_for(wl), "lanes": lanes,
                      "l2": "flushed between timed steps (256 MiB write, then 256 MiB read)",
                      "parallelism": f"time-sharded x{world}",
                      "cuda_graph": graph is not None}}

    # ---- CPU reference on a bounded prefix + parity of the same prefix
    res["cpu_sample"], res["parity"] = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        arm = CpuArm(h0, hs, dt, mode)
        target = args.cpu_seconds if headline else min(args.cpu_seconds, 4.0)
        s = arm.sample(values, target)
        res["cpu_sample"] = arm.baseline(s, n)
        u_seq = arm.run(s["prefix"], reduction="sequential")
        gpu_u = ctx.equiprop(sp.ControlAmplitudes(s["prefix"], dt)).u
        den = np.linalg.norm(s["u"])
        err = float(np.linalg.norm(gpu_u - s["u"]) / den)
        eps_self = float(np.linalg.norm(u_seq - s["u"]) / den)
        tol = max(1e-12, 4.0 * eps_self)
        res["parity"] = {"slices": s["slices"], "against": arm.kind, "rel_fro": err,
                         "eps_self": eps_self, "tol": tol, "pass": bool(err <= tol)}
        arm.close()
    ctx.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    # (the microsecond-scale qubit lines first, the seconds-long C4 magnus
    # line last: each secondary measured before the next heats the board)
    ap.add_argument("--secondary", default="c1,c1m,c3s,c3,c4m",
                    help="extra workloads reported under per_dim ('' for none)")
    ap.add_argument("--cpu-seconds", type=float, default=9.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the secondary workloads directly instead of as CUDA graphs")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # one rank per GPU; BENCH_DIST_BACKEND=gloo folds several ranks onto the
    # visible GPUs (a functional check of the multi-rank path on a 1-GPU box)
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local_rank = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    dist = None
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist_mod
        if backend == "nccl":
            dist_mod.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist_mod.init_process_group(backend)
        dist = dist_mod

    head = measure_gpu(args, args.workload, rank, world, local_rank, dist, True)
    per_dim = {}
    for name in [s for s in args.secondary.split(",") if s and s != args.workload]:
        r = measure_gpu(args, name, rank, world, local_rank, dist, False)
        per_dim[name] = {"value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"],
                         "steps": r["steps"], "e2e": r["e2e"],
                         "roofline_bound": r["roofline"]["bound"],
                         "roofline_frac": r["roofline"]["frac"],
                         "roofline_achieved": r["roofline"]["achieved"],
                         "roofline_peak": r["roofline"]["peak"],
                         "roofline_unit": r["roofline"]["unit"],
                         "pipe_frac": r["roofline"]["pipe_frac"],
                         "canonical_frac": r["roofline"]["canonical_frac"],
                         "pipe": r["roofline"]["pipe"],
                         "kernel": r["roofline"]["kernel"], "workload": r["config"]["workload"],
                         "m": r["m"], "lanes": r["lanes"], "cuda_graph": r["config"]["cuda_graph"],
                         "cpu_baseline": r["cpu_sample"], "parity": r["parity"]}
    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "complex128", "data": "synthetic (seeded random unit-norm Hermitian "
                                           "system, uniform(-1,1) amplitudes)",
            "config": head["config"], "roofline": head["roofline"],
            "cpu_baseline": head["cpu_sample"], "parity": head["parity"], "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
            "per_dim": per_dim, "impl": "b200",
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
