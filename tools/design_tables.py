"""Regenerate the measured tables of DESIGN.md §4 from profiles/.

    python tools/design_tables.py profiles/r01_bench_vN.jsonl

Rewrites the C5 sweep table (profiles/r01_sweep_c5.jsonl, complex128 at 1e6
slices, 1e4 for d >= 256) and the bench table rows (C4 headline and the
per_dim secondary lines) in place.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = 37.09


def sweep_table():
    rows = {}
    for line in open(os.path.join(ROOT, "profiles", "r01_sweep_c5.jsonl")):
        d = json.loads(line)
        if "skipped" in d or d["precision"] != "fp64":
            continue
        rows[(d["dim"], d["slices"])] = d
    out = []
    for dim in (2, 4, 8, 16, 32, 64, 128, 256, 512):
        d = rows[(dim, 1000000 if dim < 256 else 10000)]
        k = d["kernel"].replace("lane_", "").replace("_kernel", "")
        out.append(f"| {dim} | {k} | {d['slices_per_s']:.3g} | {d['fp64_roofline_frac']:.2f} | "
                   f"{d['executed_frac']:.2f} | {d['cpu_slices_per_s']:.3g} | "
                   f"{d['gpu_over_cpu']:,.0f}× |")
    return "\n".join(out)


def main():
    bench = json.loads(open(sys.argv[1]).read())
    path = os.path.join(ROOT, "DESIGN.md")
    s = open(path).read()
    a = s.index("| 2 | small<2,1> |")
    b = s.index("\n\ncomplex64 contexts run the same FP64 kernels")
    s = s[:a] + sweep_table() + s[b:]
    r, pd = bench["roofline"], bench["per_dim"]

    def row(v, key):
        return v[key]
    new = {
        "| C4 d=128": f"| C4 d=128, N=4, 1e6, m=13 (PS3g) | {bench['value']:.4g} | "
                      f"{bench['e2e']['value']:.4g} | {r['frac'] * PEAK:.1f} | {r['frac']:.2f} | "
                      f"{r['executed_frac']:.3f} | {bench['cpu_baseline']['value']:.0f} slices/s "
                      f"(oracle port) |",
        "| C3 d=32": f"| C3 d=32, N=2, 1e6, m=13 (PS) | {pd['c3']['value']:.4g} | "
                     f"{pd['c3']['e2e']['value']:.4g} | {pd['c3']['roofline_frac'] * PEAK:.1f} | "
                     f"{pd['c3']['roofline_frac']:.2f} | {pd['c3']['executed_frac']:.3f} | "
                     f"8.6e3 (sweep) |",
        "| C1 d=2": f"| C1 d=2 qubit, 1e5, m=3 (one launch) | {pd['c1']['value']:.3g} | "
                    f"{pd['c1']['e2e']['value']:.3g} | {pd['c1']['roofline_frac'] * PEAK:.2f} | "
                    f"{pd['c1']['roofline_frac']:.3f} (latency-bound, "
                    f"{pd['c1']['ms_per_step'] * 1e3:.0f} µs/step) | {pd['c1']['executed_frac']:.3f} | "
                    f"6.3e5 (sweep) |",
        "| C3 physics": f"| C3 physics variant: 5-spin chain d=32 (`SpinChain`), 1e6, m=3 (Clenshaw) | "
                        f"{pd['c3s']['value']:.3g} | {pd['c3s']['e2e']['value']:.3g} | "
                        f"{pd['c3s']['roofline_frac'] * PEAK:.1f} | {pd['c3s']['roofline_frac']:.2f} | "
                        f"{pd['c3s']['executed_frac']:.3f} | — |",
        "| north-star": f"| north-star d=2 qubit, 1e6, m=3 (one launch) | {pd['c1m']['value']:.3g} | "
                        f"{pd['c1m']['e2e']['value']:.3g} | {pd['c1m']['roofline_frac'] * PEAK:.1f} | "
                        f"{pd['c1m']['roofline_frac']:.3f} ({pd['c1m']['ms_per_step'] * 1e3:.0f} "
                        f"µs/step) | {pd['c1m']['executed_frac']:.3f} | 6.3e5 |",
    }
    lines = s.split("\n")
    for i, line in enumerate(lines):
        for k, v in new.items():
            if line.startswith(k):
                lines[i] = v
    s = "\n".join(lines)
    a = s.index("### Measured (round 1, `profiles/")
    b = s.index("`", a + len("### Measured (round 1, `"))
    s = s[:a] + "### Measured (round 1, `profiles/" + os.path.basename(sys.argv[1]) + s[b:]
    open(path, "w").write(s)
    print(sweep_table())


if __name__ == "__main__":
    main()
