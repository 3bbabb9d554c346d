"""Generate the golden fixtures from the REFERENCE implementation.

Run in the build container only (it imports the read-only reference at
/root/reference/pkg/src; the GPU box has no copy of it):

    python tests/golden/make_golden.py

Outputs (committed):
  tests/golden/plan.npz        host-plan KATs (bessel_j, chebyshev_error,
                               select_m_max, norm_capability, make_plan)
  tests/golden/equiprop.npz    small equiprop / equiprop_all cases for every
                               mode, precision and a ladder of dimensions
  tests/golden/converge.json   driven-qubit convergence sweep errors and
                               fitted orders (sliceprop.studies)

Inputs of the larger cases are regenerated from seeds by
``tests/golden/cases.py`` (shared with the tests); a SHA-256 of the
regenerated inputs is stored next to every output so drift is detected.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import sliceprop as ref  # noqa: E402  (reference, build container only)
from sliceprop import studies as ref_studies  # noqa: E402

from cases import CASES, CONVERGE_PTS, build_inputs, input_digest  # noqa: E402


def plan_fixture():
    out = {}
    ks = list(range(0, 65))
    xs = [0.0, 1e-6, 5e-5, 9.9e-5, 1e-4, 3.6e-5, 0.003, 0.05, 0.2, 0.25, 0.5, 0.9, 1.0,
          1.5, 2.0, 3.0, 4.447, 5.3, 7.5, 9.919, 16.0, 19.1, 31.0, 49.5, 64.0]
    bj = np.array([[ref.chebyshev.bessel_j(k, x) for x in xs] for k in ks])
    out["bessel_k"] = np.array(ks)
    out["bessel_x"] = np.array(xs)
    out["bessel_j"] = bj
    spans = np.concatenate([[0.0], np.logspace(-6, 1.3, 60)])
    out["err_spans"] = spans
    out["chebyshev_error"] = np.array(
        [[ref.chebyshev_error(m, s) for s in spans] for m in ref.ORDER_GRID])
    bounds = np.concatenate([[0.0], np.logspace(-7, 1.0, 80)])
    sel = np.zeros((2, bounds.size), dtype=np.int64)
    for pi, prec in enumerate(("fp32", "fp64")):
        for bi, b in enumerate(bounds):
            try:
                sel[pi, bi] = ref.select_m_max(b, ref.Precision.parse(prec))
            except ref.StepTooLargeError:
                sel[pi, bi] = -1
    out["select_bounds"] = bounds
    out["select_m"] = sel
    out["capability"] = np.array(
        [[ref.norm_capability(m, ref.Precision.parse(p)) for m in ref.ORDER_GRID]
         for p in ("fp32", "fp64")])
    betas = [0.0, 3.6e-5, 0.05, 0.5, 1.0, 1.01, 2.5, 4.4]
    coeffs = np.zeros((2, len(betas), 26), dtype=np.complex128)
    ms = np.zeros((2, len(betas)), dtype=np.int64)
    perr = np.zeros((2, len(betas)))
    for pi, prec in enumerate(("fp32", "fp64")):
        for bi, b in enumerate(betas):
            try:
                plan = ref.make_plan(-b, b, ref.Precision.parse(prec))
            except ref.StepTooLargeError:
                ms[pi, bi] = -1
                continue
            ms[pi, bi] = plan.m_max
            coeffs[pi, bi, :plan.m_max + 1] = plan.coeffs
            perr[pi, bi] = plan.predicted_error
    out["plan_betas"] = np.array(betas)
    out["plan_m"] = ms
    out["plan_coeffs"] = coeffs
    out["plan_predicted_error"] = perr
    np.savez_compressed(os.path.join(HERE, "plan.npz"), **out)


def run_reference(case, h0, hs, values, dt):
    mode = case["mode"]
    ctx = ref.create(precision=case["precision"], m_max=case.get("m_max"))
    magnus = mode == "magnus"
    quad = None if magnus else mode
    ctx.set_hamiltonian(ref.ControlSystem(h0, hs), magnus=magnus, quadrature=quad)
    amps = ref.ControlAmplitudes(values, dt)
    pair = ctx.equiprop(amps, reduction="pairwise")
    seq = ctx.equiprop(amps, reduction="sequential")
    res = {"u": pair.u, "u_seq": seq.u, "slice_count": pair.slice_count}
    if pair.plan is not None:
        res.update({"beta": pair.plan["beta"], "m_max": pair.plan["m_max"],
                    "predicted_error": pair.plan["predicted_error"]})
    if case.get("cumulative"):
        res["u_all"] = ctx.equiprop_all(amps).u_all
    ctx.close()
    return res


def equiprop_fixture():
    out = {}
    names = []
    for case in CASES:
        h0, hs, values, dt = build_inputs(case)
        res = run_reference(case, h0, hs, values, dt)
        key = case["name"]
        names.append(key)
        out[f"{key}__digest"] = np.frombuffer(input_digest(h0, hs, values, dt), dtype=np.uint8)
        for k, v in res.items():
            out[f"{key}__{k}"] = np.asarray(v)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "equiprop.npz"), **out)


def converge_fixture():
    problem = ref_studies.DrivenQubit(1.0, 0.1, 1.0, 6.0)
    res = {}
    for label, magnus, quad, prec in [("midpoint", False, "midpoint", "fp64"),
                                      ("simpson", False, "simpson", "fp64"),
                                      ("magnus", True, None, "fp64"),
                                      ("magnus_fp32", True, None, "fp32")]:
        rows = ref_studies.convergence_sweep(problem, CONVERGE_PTS, magnus=magnus,
                                             quadrature=quad, precision=prec)
        pts = [p for p, _ in rows]
        errs = [e for _, e in rows]
        entry = {"pts": pts, "errors": errs}
        try:
            order, window = ref_studies.fit_convergence_order(pts, errs)
            entry["order"] = order
            entry["window"] = list(window)
        except ValueError:
            entry["order"] = None
        res[label] = entry
    res["exact"] = [[z.real, z.imag] for z in problem.exact_propagator().ravel()]
    with open(os.path.join(HERE, "converge.json"), "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    plan_fixture()
    equiprop_fixture()
    converge_fixture()
    for f in ("plan.npz", "equiprop.npz", "converge.json"):
        p = os.path.join(HERE, f)
        print(f, os.path.getsize(p), hashlib.sha256(open(p, "rb").read()).hexdigest()[:16])
