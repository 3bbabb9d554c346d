"""equiprop_all on one B200: device-resident cumulative
propagators, the HBM-write-bound path, against the measured HBM bandwidth.

    python tools/cum_bench.py [--out gpurun_out/cum.jsonl]

bytes/slice (algorithmic) = d^2 * 16 (the complex128 output); the kernels also
write and re-read the in-lane prefixes (2 * D^2 * 16, D the padded family
size), reported as "traffic_est".  Times: CUDA events around the device entry
(lane kernel + fold + prefix application), median of 3 after a warm-up.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

CASES = [(2, 4_000_000), (4, 2_000_000), (8, 1_000_000), (16, 400_000), (32, 100_000),
         (64, 20_000), (128, 4_000), ("qubit", 4_000_000)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cum.jsonl"))
    ap.add_argument("--dims", default="", help="comma-separated subset of the case dims")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cases = [c for c in CASES if not a.dims or str(c[0]) in a.dims.split(",")]
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import torch

    import paper_2108_07126_b200 as sp
    from cases import unit_hermitian
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6533.0
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    fh = open(a.out, "w")
    for d, n in cases:
        label = d
        if d == "qubit":  # the driven qubit: su(2) lanes in the two-pass form
            from cases import qubit_inputs
            h0, hs, values, dt = qubit_inputs(n, "midpoint")
            d = 2
        else:
            rng = np.random.default_rng(20240911)
            h0 = unit_hermitian(rng, d)
            hs = [unit_hermitian(rng, d) for _ in range(2)]
            values = rng.uniform(-1.0, 1.0, (n, 2))
            dt = 0.5 / 3.0
        ctx = sp.create()
        ctx.set_hamiltonian(sp.ControlSystem(h0, hs))
        plan = ctx.plan_for(dt)
        d_amps = torch.from_numpy(values).to(dev)
        out = torch.empty((n, d, d), dtype=torch.complex128, device=dev)
        run = lambda: ctx.equiprop_all_device_ptr(d_amps.data_ptr(), n, 2, dt, out.data_ptr(),
                                                  stream=stream.cuda_stream, plan=plan)
        run()
        torch.cuda.synchronize(dev)
        ms = []
        for _ in range(a.reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms.append(e0.elapsed_time(e1))
        t = statistics.median(ms) / 1e3
        D = {2: 2, 4: 4, 8: 8}.get(d, d)
        out_b = n * d * d * 16
        est = out_b + 2 * n * D * D * 16
        rec = {"dim": d, "system": "driven qubit" if label == "qubit" else "random",
               "kernel": ctx.last_timing()["kernel"], "slices": n, "ms": t * 1e3,
               "slices_per_s": n / t,
               "output_gb_s": out_b / t / 1e9, "traffic_est_gb_s": est / t / 1e9,
               "hbm_frac_output": out_b / t / 1e9 / hbm, "hbm_frac_traffic_est": est / t / 1e9 / hbm,
               "output_bytes": out_b, "hbm_gbs_peak": hbm}
        print(json.dumps(rec), flush=True)
        fh.write(json.dumps(rec) + "\n")
        ctx.close()
        del out, d_amps
        torch.cuda.empty_cache()
    fh.close()


if __name__ == "__main__":
    main()
