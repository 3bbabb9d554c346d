"""C2 (BASELINE.json configs[1]): the driven-qubit dt convergence sweep on the
B200 path next to the reference's own golden errors.

    python tools/c2_converge.py [--out profiles/r01_converge_c2.md]

Runs convergence_sweep (studies.py, the reference's `sliceprop converge`
protocol: max|U - U_exact| against the analytic propagator) for midpoint,
simpson and magnus in complex128 and magnus in complex64 over the
reference's DEFAULT_SWEEP, prints each error beside the reference's, and
fits the convergence order over the reference's windows.
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2108_07126_b200.studies import (DrivenQubit, convergence_sweep,  # noqa: E402
                                           fit_convergence_order)

SWEEP = [10, 32, 100, 316, 1000, 3162, 10000, 31623, 100000, 316228, 1000000]
# reference goldens (`python3 -m sliceprop converge`)
REF = {
    "midpoint c128": [4.284213033727e-03, 4.196847558336e-04, 4.298866541365e-05,
                      4.305198906730e-06, 4.299012879318e-07, 4.299762990626e-08,
                      4.298989482923e-09, 4.297489747538e-10, 4.541581356902e-11,
                      1.895445098049e-11, 9.662819410428e-11],
    "simpson c128": [3.277722459904e-02, 3.342984002081e-03, 3.437571322846e-04,
                     3.444006468721e-05, 3.439194954338e-06, 3.439813457554e-07,
                     3.439210081595e-08, 3.439313252172e-09, 3.432316302781e-10,
                     3.283457579522e-11, 9.053930412639e-12],
    "magnus c128": [2.128645483030e-03, 2.137034966001e-05, 2.252084784818e-07,
                    2.259747030503e-09, 2.253378056547e-11, 2.210133665658e-13,
                    4.220746132047e-14, 5.989512380445e-13, 2.248054918670e-12,
                    1.237322784785e-11, 4.600961068841e-11],
    "magnus c64": [2.128628068242e-03, 2.134823614354e-05, 2.195857610443e-06,
                   5.684051965162e-06, 5.693609068497e-07, 3.845041185343e-05,
                   4.751451640012e-05, 1.723891389893e-04, 3.803713286025e-04,
                   3.461374546649e-04, 2.393564820448e-04],
}
RUNS = {"midpoint c128": dict(magnus=False, quadrature="midpoint", precision="fp64"),
        "simpson c128": dict(magnus=False, quadrature="simpson", precision="fp64"),
        "magnus c128": dict(magnus=True, quadrature=None, precision="fp64"),
        "magnus c64": dict(magnus=True, quadrature=None, precision="fp32"),
        # extensions (no reference rows): 4th-order Gauss-Legendre Magnus and
        # the 2-node average, same sample counts (coerced even)
        "gauss-legendre magnus c128": dict(magnus=True, quadrature="gauss-legendre",
                                           precision="fp64"),
        "gauss-legendre average c128": dict(magnus=False, quadrature="gauss-legendre",
                                            precision="fp64")}
BANDS = {"midpoint c128": (1.9, 2.2), "simpson c128": (1.9, 2.2), "magnus c128": (3.7, 4.3),
         "gauss-legendre magnus c128": (3.7, 4.3), "gauss-legendre average c128": (1.9, 2.2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "converge_c2.md"))
    a = ap.parse_args()
    q = DrivenQubit(1.0, 0.1, 1.0, 6.0)
    out = ["# C2: driven-qubit dt convergence on one B200 vs the reference (sliceprop 0.1.0)",
           "", "error = max|U - U_exact| (analytic propagator); reference = BASELINE.md §4 goldens",
           ""]
    for name, kw in RUNS.items():
        t0 = time.perf_counter()
        rows = convergence_sweep(q, SWEEP, **kw)
        sec = time.perf_counter() - t0
        pts = [p for p, _ in rows]
        err = [e for _, e in rows]
        out += [f"## {name}  ({sec:.1f} s for the whole sweep)", "",
                "| pts | B200 error | reference error | ratio |", "|---|---|---|---|"]
        ref_rows = REF.get(name, REF["magnus c128"] if "magnus" in name else REF["midpoint c128"])
        if name not in REF:
            out[-1:] = ["| pts | B200 error | reference error (Simpson-Magnus / midpoint, "
                        "nearest pts) | ratio |", "|---|---|---|---|"]
        for p, e, r in zip(pts, err, ref_rows):
            out.append(f"| {p} | {e:.6e} | {r:.6e} | {e / r:.4f} |")
        if name in BANDS:
            order, (lo, hi) = fit_convergence_order(pts, err)
            ref_order, _ = fit_convergence_order(pts, ref_rows)
            band = BANDS[name]
            ok = band[0] <= order <= band[1]
            out += ["", f"fitted order {order:.4f} over pts {lo}..{hi} (reference {ref_order:.4f}; "
                        f"acceptance band {band}: {'inside' if ok else 'OUTSIDE'})"]
        out.append("")
    text = "\n".join(out)
    print(text)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write(text + "\n")


if __name__ == "__main__":
    main()
