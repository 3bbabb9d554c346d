"""Seeded parity cases shared by the golden generator and the tests.

Every case is regenerated bit-identically from its description (numpy's
PCG64 ``default_rng`` and closed-form drives), so the fixture only needs to
store the reference OUTPUTS plus a digest of the inputs.

Problem families (reference anchors):
  qubit   the circularly driven qubit of the paper, ``studies.py:51-90``
  random  unit 1-norm random Hermitian drift/controls as in ``bench_grid``
          (``studies.py:248-283``), dt = beta_target / sum of 1-norms
  zero    zero Hamiltonian (exact identity, ``test_propagator.py:251-255``)
"""

from __future__ import annotations

import hashlib

import numpy as np

SEED = 20240911  # reference conftest.py:5-7, studies.py:257

PAULI_X = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)
PAULI_Y = np.array([[0.0, -1.0j], [1.0j, 0.0]], dtype=complex)
PAULI_Z = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=complex)

# sliceprop cli.py:21-22 DEFAULT_SWEEP truncated at 1e5 to keep the
# generator and the GPU test quick
CONVERGE_PTS = [10, 32, 100, 316, 1000, 3162, 10000, 31623, 100000]


def unit_hermitian(rng, d):
    a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    h = 0.5 * (a + a.conj().T)
    return h / np.abs(h).sum(axis=0).max()


def qubit_inputs(pts, mode, w0=1.0, w1=0.1, wrf=1.0, duration=6.0):
    """DrivenQubit(1, 0.1, 1, 6) system + samples (``studies.py:51-90``)."""
    h0 = 0.5 * w0 * PAULI_Z
    hs = [0.5 * w1 * PAULI_X, 0.5 * w1 * PAULI_Y]
    if mode == "midpoint":
        dt = duration / max(pts, 1)
        t = (np.arange(pts) + 0.5) * dt
    else:
        dt = duration / (pts - 1)
        t = np.arange(pts) * dt
    values = np.column_stack([np.cos(wrf * t), np.sin(wrf * t)])
    return h0, hs, values, dt


def random_inputs(d, n_ctrl, pts, seed, beta=0.5):
    rng = np.random.default_rng(seed)
    h0 = unit_hermitian(rng, d)
    hs = [unit_hermitian(rng, d) for _ in range(n_ctrl)]
    dt = beta / (n_ctrl + 1.0)
    values = rng.uniform(-1.0, 1.0, (pts, n_ctrl))
    return h0, hs, values, dt


def build_inputs(case):
    kind = case["kind"]
    if kind == "qubit":
        return qubit_inputs(case["pts"], case["mode"])
    if kind == "random":
        return random_inputs(case["d"], case["n_ctrl"], case["pts"],
                             case.get("seed", SEED), case.get("beta", 0.5))
    if kind == "zero":
        d = case["d"]
        return np.zeros((d, d), dtype=complex), [], np.zeros((case["pts"], 0)), 0.3
    raise ValueError(kind)


def input_digest(h0, hs, values, dt) -> bytes:
    h = hashlib.sha256()
    for m in (h0, *hs):
        h.update(np.ascontiguousarray(m, dtype=np.complex128).tobytes())
    h.update(np.ascontiguousarray(values, dtype=np.float64).tobytes())
    h.update(np.float64(dt).tobytes())
    return h.digest()


def _c(name, kind, mode, pts, precision="fp64", **kw):
    return dict(name=name, kind=kind, mode=mode, pts=pts, precision=precision, **kw)


CASES = []
# the paper's driven qubit (config C1/C2 shapes at small n)
for pts in (1, 2, 7, 100, 1000):
    CASES.append(_c(f"qubit_mid_{pts}", "qubit", "midpoint", pts))
CASES.append(_c("qubit_mid_12_cum", "qubit", "midpoint", 12, cumulative=True))
for pts in (3, 101, 1001):
    CASES.append(_c(f"qubit_simpson_{pts}", "qubit", "simpson", pts))
    CASES.append(_c(f"qubit_magnus_{pts}", "qubit", "magnus", pts))
CASES.append(_c("qubit_mid_100_fp32", "qubit", "midpoint", 100, "fp32"))
CASES.append(_c("qubit_magnus_101_fp32", "qubit", "magnus", 101, "fp32"))
CASES.append(_c("zero_d2", "zero", "midpoint", 6, d=2))
# random unit-norm systems: dimension ladder x modes (incl. non powers of two)
for d in (1, 2, 3, 4, 5, 8, 12, 16, 24, 32):
    CASES.append(_c(f"rand_d{d}_mid", "random", "midpoint", 33, d=d, n_ctrl=2, seed=SEED + d))
    CASES.append(_c(f"rand_d{d}_simpson", "random", "simpson", 33, d=d, n_ctrl=2,
                    seed=SEED + 100 + d))
    CASES.append(_c(f"rand_d{d}_magnus", "random", "magnus", 33, d=d, n_ctrl=2,
                    seed=SEED + 200 + d))
CASES.append(_c("rand_d3_drift_only", "random", "midpoint", 5, d=3, n_ctrl=0, seed=7))
CASES.append(_c("rand_d6_n3_mid", "random", "midpoint", 20, d=6, n_ctrl=3, seed=11))
CASES.append(_c("rand_d4_n3_magnus_cum", "random", "magnus", 17, d=4, n_ctrl=3, seed=12,
                cumulative=True))
CASES.append(_c("rand_d32_mid_cum", "random", "midpoint", 10, d=32, n_ctrl=2, seed=13,
                cumulative=True))
CASES.append(_c("rand_d8_cap_edge", "random", "midpoint", 9, d=8, n_ctrl=2, seed=14, beta=4.4))
CASES.append(_c("rand_d4_mmax25", "random", "midpoint", 9, d=4, n_ctrl=1, seed=15, m_max=25))
CASES.append(_c("rand_d4_mmax5", "random", "midpoint", 9, d=4, n_ctrl=1, seed=16, m_max=5,
                beta=0.05))
for d in (2, 8, 32):
    CASES.append(_c(f"rand_d{d}_mid_fp32", "random", "midpoint", 33, "fp32", d=d, n_ctrl=2,
                    seed=SEED + 300 + d))
    CASES.append(_c(f"rand_d{d}_magnus_fp32", "random", "magnus", 33, "fp32", d=d,
                    n_ctrl=2, seed=SEED + 400 + d))
CASES.append(_c("rand_d64_mid", "random", "midpoint", 16, d=64, n_ctrl=2, seed=SEED + 64))
CASES.append(_c("rand_d128_mid", "random", "midpoint", 8, d=128, n_ctrl=4, seed=SEED + 128))
CASES.append(_c("rand_d128_magnus", "random", "magnus", 9, d=128, n_ctrl=4,
                seed=SEED + 129))
CASES.append(_c("rand_d128_mid_fp32", "random", "midpoint", 8, "fp32", d=128, n_ctrl=4,
                seed=SEED + 130))
CASES.append(_c("rand_d48_simpson", "random", "simpson", 11, d=48, n_ctrl=3, seed=SEED + 48))

CASE_BY_NAME = {c["name"]: c for c in CASES}
assert len(CASE_BY_NAME) == len(CASES)
