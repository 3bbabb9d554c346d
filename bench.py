#!/usr/bin/env python
"""Benchmark of the equiprop hot path on B200 (contract: see DESIGN.md §Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)

Headline workload (BASELINE.json configs[3], the largest single-GPU config):
C4 = dim-128 random unit-1-norm system, 4 controls, 1e6 slices, midpoint,
complex128, beta = 0.5 (m = 13), time-sharded over the N GPUs (strong
scaling: 1e6 slices in total).  Secondary lines (same JSON, "per_dim"): C3
(dim 32, 2 controls, 1e6 slices; random and the coupled-spin chain of
configs[2]), C1 (the paper's driven qubit, dim 2,
1e5 slices) and c1m (the same qubit at the north star's 1e6 slices).
A step is one full propagation U = U_{n-1} ... U_0 of the workload; value = slices / device time (CUDA events, max over ranks), with
the amplitude table resident in HBM and L2 flushed between timed steps.
e2e = the same through the public API with the table in page-locked host
memory (H2D + kernels + gather + D2H inside the timed region, wall clock,
max over ranks).

--impl reference times the reference algorithm on the host cores: the CPU
oracle (oracle/, a bit-exact numpy restatement of sliceprop 0.1.0, which
itself cannot travel to the GPU box) on a bounded prefix of the same
workload, extrapolated linearly (runtime linear in slices is a reference
property, test_acceptance.py:229-245).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time slices/sec (complex128) at dim 2/32/128, 1/2/4/8 B200; % FP64 roofline"
UNIT = "slices/s"
SEED = 20240911

WORKLOADS = {
    "c4": dict(d=128, n_ctrl=4, slices=1_000_000, kind="random",
               label="C4: dim-128 random unit-norm system, 4 controls, 1e6 slices, midpoint, "
                     "complex128, beta=0.5 (m=13)"),
    "c3": dict(d=32, n_ctrl=2, slices=1_000_000, kind="random",
               label="C3: dim-32 random unit-norm system, 2 controls, 1e6 slices, midpoint, "
                     "complex128, beta=0.5 (m=13)"),
    "c3s": dict(d=32, n_ctrl=2, slices=1_000_000, kind="spin",
                label="C3 physics variant: 5-spin coupled chain (d=32, 2 controls, "
                      "cos/sin drive over T=6), 1e6 slices, midpoint, complex128"),
    "c1": dict(d=2, n_ctrl=2, slices=100_000, kind="qubit",
               label="C1: paper's driven qubit (w0=1, w1=0.1, wrf=1, T=6), dim 2, 2 controls, "
                     "1e5 slices, midpoint, complex128 (m=3)"),
    "c1m": dict(d=2, n_ctrl=2, slices=1_000_000, kind="qubit",
                label="north-star d=2 target: the driven qubit at 1e6 slices, midpoint, "
                      "complex128 (m=3)"),
}


def fp64_peak():
    with open(os.path.join(ROOT, "profiles", "fp64_peak.json")) as fh:
        return json.load(fh)


def make_problem(wl):
    """(system, amplitude table, dt) — deterministic synthetic inputs."""
    import paper_2108_07126_b200 as sp
    if wl["kind"] == "qubit":
        q = sp.DrivenQubit(1.0, 0.1, 1.0, 6.0)
        amps = q.amplitudes(wl["slices"])
        return q.system(), np.ascontiguousarray(amps.values), amps.dt
    if wl["kind"] == "spin":
        c = sp.SpinChain()
        amps = c.amplitudes(wl["slices"])
        return c.system(), np.ascontiguousarray(amps.values), amps.dt
    rng = np.random.default_rng(SEED)
    from paper_2108_07126_b200.studies import random_system
    system = random_system(rng, wl["d"], wl["n_ctrl"])
    dt = 0.5 / sum(system.norms)
    values = rng.uniform(-1.0, 1.0, (wl["slices"], wl["n_ctrl"]))
    return system, values, dt


def canonical_flops(d, m, n_terms):
    """F(d, m, T) = 8 d^3 (m + 1) + 4 d^2 T per slice."""
    return 8.0 * d ** 3 * (m + 1) + 4.0 * d * d * n_terms


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


def cpu_sample_rate(system, values, dt, target_s=8.0, max_slices=50_000):
    """Oracle (reference algorithm, numpy/OpenBLAS, all host threads) on a
    bounded prefix; returns (slices/s, slices timed, seconds, threads)."""
    import oracle
    h0, hs = system.drift, list(system.controls)
    n0 = 64 if system.dim >= 64 else 4096
    oracle.equiprop(h0, hs, values[:n0 // 4], dt, mode="midpoint")  # warm BLAS threads
    t0 = time.perf_counter()
    oracle.equiprop(h0, hs, values[:n0], dt, mode="midpoint")
    per = (time.perf_counter() - t0) / n0
    n = int(max(n0, min(max_slices, values.shape[0], target_s / max(per, 1e-9))))
    t0 = time.perf_counter()
    oracle.equiprop(h0, hs, values[:n], dt, mode="midpoint")
    sec = time.perf_counter() - t0
    return n / sec, n, sec, blas_threads()


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()
                    if i.get("user_api") == "blas"), default=1)
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    """--impl reference: rank 0 times the reference algorithm on the host."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    wl = WORKLOADS[args.workload]
    system, values, dt = make_problem(wl)
    import oracle
    h0, hs = system.drift, list(system.controls)
    _, n, sec, threads = cpu_sample_rate(system, values, dt, target_s=args.cpu_seconds)
    for _ in range(args.warmup):
        oracle.equiprop(h0, hs, values[:max(1, n // 4)], dt, mode="midpoint")
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.equiprop(h0, hs, values[:n], dt, mode="midpoint")
        times.append(time.perf_counter() - t0)
    rate = n / statistics.median(times)
    per_step_full_ms = wl["slices"] / rate * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step_full_ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "complex128", "data": "synthetic",
        "config": {"workload": wl["label"], "dim": wl["d"], "n_ctrl": wl["n_ctrl"],
                   "slices": wl["slices"], "mode": "midpoint",
                   "sample_slices_per_step": n,
                   "note": "ms_per_step extrapolated linearly from the sample"},
        "cpu_baseline": {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"first {n} slices of the workload per step, median of "
                                   f"{args.steps} steps, oracle/ numpy restatement of the "
                                   f"reference (OpenBLAS {threads} threads, host "
                                   f"{os.cpu_count()} cpus)"},
        "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def max_over_ranks(dist, vals, dev):
    import torch
    on = dev if dist.get_backend() == "nccl" else "cpu"
    red = torch.tensor(vals, dtype=torch.float64, device=on)
    dist.all_reduce(red, op=dist.ReduceOp.MAX)
    return red.tolist()


def measure_gpu(args, wl, rank, world, local_rank, dist, headline):
    import torch

    import paper_2108_07126_b200 as sp
    from paper_2108_07126_b200.sharding import (equiprop_sharded_device, partition,
                                                shard_rows)
    system, values, dt = make_problem(wl)
    d, n = system.dim, values.shape[0]
    ctx = sp.create(device=local_rank)
    ctx.set_hamiltonian(system)
    ctx.set_profiling(True)
    plan = ctx.plan_for(dt)
    a, b = partition(n, world)[rank]
    lo, hi = shard_rows("midpoint", a, b)
    local = np.ascontiguousarray(values[lo:hi])
    dev = torch.device("cuda", local_rank)
    d_amps = torch.from_numpy(local).to(dev)
    out = torch.empty((d, d), dtype=torch.complex128, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > L2
    stream = torch.cuda.current_stream(dev)

    # amplitude validation (|c| <= 1) is part of the job: it runs inside the
    # lane kernel and its flag is read after each timed step (sp_amplitude_violation)
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
    # launch-latency-bound secondary workloads (C1: ~10 us of GPU work per
    # step) replay the step as a CUDA graph, the way a serving loop would;
    # the headline step (seconds of GPU work) is launched directly
    graph = None
    if world == 1 and not headline and not args.no_graph:
        try:
            ctx.set_profiling(False)
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=cap):
                ctx.equiprop_device_ptr(d_amps.data_ptr(), hi - lo, wl["n_ctrl"], dt,
                                        out.data_ptr(), stream=cap.cuda_stream, plan=plan)
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
           for _ in range(args.steps)]
    kernel_ms, launches = [], 0
    with Clocks(local_rank) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step()
            evs[k][1].record(stream)
            if graph is not None:
                stream.synchronize()
                launches += launches_per_step
            else:
                t = ctx.last_timing()
                kernel_ms.append(t["main_kernel_ms"])
                launches += t["launches"]
            validate()
        torch.cuda.synchronize(dev)
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
    value = n * args.steps / (total_ms / 1e3)
    local_slices = b - a
    F = canonical_flops(d, plan.m_max, 1 + wl["n_ctrl"])
    peak = fp64_peak()["fp64_dmma_tflops"] * 1e12
    achieved = local_slices * F / (kern / 1e3)
    traffic, traffic_note = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            cap = json.load(fh).get(t["kernel"])
        if cap:
            traffic = cap["dram_bytes"] * local_slices / cap["slices"]
            traffic_note = (f"ncu --set full dram read+write of one launch at {cap['slices']} "
                            f"slices ({cap['dram_bytes']:.3g} B), scaled linearly to this launch; "
                            f"algorithmic bytes/slice = {8 * wl['n_ctrl']} (amplitude row)")
    except (OSError, ValueError, KeyError):
        pass
    roofline = {"bound": "tensor", "achieved": achieved / 1e12, "peak": peak / 1e12,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "traffic_note": traffic_note,
                "kernel": t["kernel"], "kernel_ms": kern,
                "executed_frac": t["executed_flops"] / (kern / 1e3) / peak,
                "series": ctx.last_algorithm(),
                "algorithmic_flops_per_launch": local_slices * F,
                "peak_source": "measured FP64 DMMA pipe peak (profiles/fp64_peak.json)"}

    # ---- e2e: public API, page-locked host table, H2D + compute + D2H timed
    pinned = torch.empty(local.shape, dtype=torch.float64, pin_memory=True)
    pinned.numpy()[:] = local
    e2e_times = []
    amps_obj = sp.ControlAmplitudes(pinned.numpy(), dt, copy=False) if world == 1 else None
    for k in range(args.warmup + args.steps):
        flush.fill_(float(k))
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
    e2e = {"value": n * args.steps / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": int(local.nbytes), "d2h_bytes_per_step": int(d * d * 16),
           "ms_per_step": e2e_s / args.steps * 1e3}
    assert np.all(np.isfinite(u))
    res = {"value": value, "ms_per_step": total_ms / args.steps, "roofline": roofline,
           "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
           "m": plan.m_max, "config": {"workload": wl["label"], "dim": d,
                                       "n_ctrl": wl["n_ctrl"], "slices": n,
                                       "mode": "midpoint", "m": plan.m_max,
                                       "l2": "flushed between timed steps (256 MiB write)",
                                       "parallelism": f"time-sharded x{world}",
                                       "cuda_graph": graph is not None}}
    res["cpu_sample"] = None
    if headline and rank == 0 and world == 1 and not args.no_cpu:
        rate, ns, sec, threads = cpu_sample_rate(system, values, dt, target_s=args.cpu_seconds)
        res["cpu_sample"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"first {ns} slices of the workload ({sec:.1f} s), "
                                       "oracle/ numpy restatement of the reference, OpenBLAS "
                                       f"{threads} threads on {os.cpu_count()} host cpus"}
    ctx.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--secondary", default="c3,c3s,c1,c1m",
                    help="extra workloads reported under per_dim ('' for none)")
    ap.add_argument("--cpu-seconds", type=float, default=8.0)
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

    head = measure_gpu(args, WORKLOADS[args.workload], rank, world, local_rank, dist, True)
    per_dim = {}
    for name in [s for s in args.secondary.split(",") if s and s != args.workload]:
        r = measure_gpu(args, WORKLOADS[name], rank, world, local_rank, dist, False)
        per_dim[name] = {"value": r["value"], "unit": UNIT, "ms_per_step": r["ms_per_step"],
                         "e2e": r["e2e"], "roofline_frac": r["roofline"]["frac"],
                         "executed_frac": r["roofline"]["executed_frac"],
                         "kernel": r["roofline"]["kernel"], "workload": r["config"]["workload"],
                         "cuda_graph": r["config"]["cuda_graph"]}
    if rank == 0:
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "complex128", "data": "synthetic (seeded random unit-norm Hermitian "
                                           "system, uniform(-1,1) amplitudes)",
            "config": head["config"], "roofline": head["roofline"],
            "cpu_baseline": head["cpu_sample"], "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"], "clocks": head["clocks"],
            "per_dim": per_dim, "impl": "b200",
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
