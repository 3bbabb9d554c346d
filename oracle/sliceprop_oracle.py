"""CPU oracle: a numpy restatement of the reference ``equiprop`` hot path.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Nothing in the
product package imports this module.

Every function restates the reference algorithm with the same numpy
operation sequence, so its outputs agree with the reference bit for bit
(pinned by ``tests/test_oracle.py`` against the fixtures that
``tests/golden/make_golden.py`` produced from the reference itself).
Reference = ``/root/reference/pkg/src/sliceprop`` (sliceprop 0.1.0).

Layout conventions (reference ``linalg.py:1-13``): complex matrices are
row-major, interleaved re/im (numpy complex128/complex64), a batch is an
``(n, d, d)`` array.  The time order is U = U[n-1] ... U[0], later slice on
the left (``propagator.py:68-80``).
"""

from __future__ import annotations

import cmath
import math

import numpy as np

__all__ = [
    "ORDER_GRID",
    "roundoff",
    "complex_dtype",
    "real_dtype",
    "bessel_j",
    "chebyshev_error",
    "select_m_max",
    "norm_capability",
    "make_plan",
    "one_norm",
    "commutator",
    "effective_terms",
    "slice_table",
    "gauss_table",
    "spectral_bound",
    "expand",
    "expm_clenshaw",
    "reduce_pairwise",
    "reduce_sequential",
    "cumulative",
    "slice_propagators",
    "equiprop",
    "equiprop_all",
    "midpoint_reference_ld",
    "StepTooLarge",
]

# chebyshev.py:50-51 — odd truncation orders 3..25
ORDER_GRID = tuple(range(3, 26, 2))
_MAX_TRUSTED_S = 1.0 / math.sqrt(2.0)          # chebyshev.py:56
_EXPM_CHUNK_BYTES = 1 << 22                     # propagator.py:125-129
_GEMM_BLOCK_BYTES = 1 << 23                     # linalg.py:201-202


class StepTooLarge(Exception):
    """Oracle-side stand-in for the reference StepTooLargeError
    (``errors.py:72-86``)."""

    def __init__(self, norm_bound, capability):
        super().__init__(f"norm bound {norm_bound} exceeds capability {capability}")
        self.norm_bound = norm_bound
        self.capability = capability


def roundoff(bits: int) -> float:
    """Unit roundoff of the working precision (``linalg.py:52-55``)."""
    return 2.0 ** -24 if bits == 32 else 2.0 ** -53


def complex_dtype(bits: int):
    return np.dtype(np.complex64 if bits == 32 else np.complex128)


def real_dtype(bits: int):
    return np.dtype(np.float32 if bits == 32 else np.float64)


# --------------------------------------------------------------------------
# host plan (chebyshev.py:61-218)
# --------------------------------------------------------------------------

def bessel_j(k: int, x: float) -> float:
    """J_k(x), 0<=k<=64, 0<=x<=64: Miller backward recurrence in 80-bit
    extended precision normalised by J_0 + 2 sum J_2j = 1
    (``chebyshev.py:61-104``)."""
    x = float(x)
    if x == 0.0:
        return 1.0 if k == 0 else 0.0
    if x < 1e-4:                                   # chebyshev.py:77-80
        half = 0.5 * x
        y = half ** 2
        head = 1.0 - y / (k + 1) + y * y / (2.0 * (k + 1) * (k + 2))
        return half ** k / math.factorial(k) * head
    top = max(k, math.ceil(x)) + 52                # chebyshev.py:82-83
    top += top % 2
    L = np.longdouble
    xl = L(x)
    below, cur = L(0.0), L(1e-30)
    even_sum = L(2.0) * cur
    picked = cur if k == top else L(0.0)
    for n in range(top, 0, -1):                    # chebyshev.py:92-103
        below, cur = cur, (L(2 * n) / xl) * cur - below
        order = n - 1
        if order == k:
            picked = cur
        if order > 0 and order % 2 == 0:
            even_sum += L(2.0) * cur
        if abs(cur) > 1e250:
            below *= L(1e-250)
            cur *= L(1e-250)
            even_sum *= L(1e-250)
            picked *= L(1e-250)
    return float(picked / (even_sum + cur))


def chebyshev_error(m: int, span: float) -> float:
    """4 (e^{1-s^2} s)^{m+1}, s = span/(4m+4) (``chebyshev.py:107-110``)."""
    s = span / (4.0 * m + 4.0)
    return 4.0 * (math.exp(1.0 - s * s) * s) ** (m + 1)


def norm_capability(m: int, bits: int) -> float:
    """Bisection for the largest g with eps(m, 2g) <= u (``chebyshev.py:137-152``)."""
    target = roundoff(bits)
    lo, hi = 0.0, (4.0 * m + 4.0) * _MAX_TRUSTED_S / 2.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if chebyshev_error(m, 2.0 * mid) <= target:
            lo = mid
        else:
            hi = mid
        if hi - lo <= 1e-15 * hi:
            break
    return 0.5 * (lo + hi)


def select_m_max(norm_bound: float, bits: int) -> int:
    """Smallest odd m meeting the roundoff target (``chebyshev.py:113-134``)."""
    span = 2.0 * norm_bound
    target = roundoff(bits)
    for m in ORDER_GRID:
        if span / (4.0 * m + 4.0) > _MAX_TRUSTED_S:
            continue
        if chebyshev_error(m, span) <= target:
            return m
    raise StepTooLarge(norm_bound, norm_capability(ORDER_GRID[-1], bits))


def make_plan(alpha: float, beta: float, bits: int, m_max=None) -> dict:
    """Plan dict {alpha, beta, m_max, coeffs, phase, predicted_error}
    (``chebyshev.py:185-218``)."""
    alpha, beta = float(alpha), float(beta)
    span = beta - alpha
    if m_max is None:
        m_max = select_m_max(span / 2.0, bits)
    else:
        eps = chebyshev_error(m_max, span)
        if span > 4.0 * m_max + 4.0 or eps >= 1.0:
            raise StepTooLarge(span / 2.0, norm_capability(m_max, bits))
    half = span / 2.0
    coeffs = np.array([(-1j) ** k * bessel_j(k, half) for k in range(m_max + 1)],
                      dtype=np.complex128)
    return {"alpha": alpha, "beta": beta, "m_max": m_max, "coeffs": coeffs,
            "phase": cmath.exp(-0.5j * (alpha + beta)),
            "predicted_error": chebyshev_error(m_max, span)}


# --------------------------------------------------------------------------
# system model (hamiltonian.py:156-207, magnus.py:36-141)
# --------------------------------------------------------------------------

def one_norm(m) -> float:
    """Largest absolute column sum (``linalg.py:313-318``)."""
    return float(np.abs(np.asarray(m)).sum(axis=0).max())


def commutator(a, b) -> np.ndarray:
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return a @ b - b @ a                         # magnus.py:36-42


def effective_terms(h0, hs, magnus: bool):
    """Expansion terms and the 1-norm groups for the bound.

    midpoint/simpson: [H0, H1..HN]; magnus: [H0, H1..HN, i[H0,Hk].., i[Hk,Hk']..]
    (``magnus.py:45-85``).  Returns (terms, base_norms, drift_comm_norms,
    cross_comm_norms)."""
    h0 = np.asarray(h0, dtype=np.complex128).copy()
    hs = [np.asarray(h, dtype=np.complex128).copy() for h in hs]
    base_norms = [one_norm(h) for h in (h0, *hs)]
    if not magnus:
        return [h0, *hs], base_norms, [], []
    n = len(hs)
    dcomm = [commutator(h0, hs[k]) for k in range(n)]
    ccomm = [commutator(hs[k], hs[kp]) for k in range(n) for kp in range(k + 1, n)]
    terms = [h0, *hs, *(1j * c for c in dcomm), *(1j * c for c in ccomm)]
    return (terms, base_norms, [one_norm(c) for c in dcomm],
            [one_norm(c) for c in ccomm])


def slice_table(values: np.ndarray, dt: float, mode: str):
    """(table, scale, slice_count) with column 0 = 1 (drift weight).

    midpoint ``hamiltonian.py:199-201``; simpson ``:202-205`` with
    ``simpson_triplets`` ``:177-183``; magnus ``magnus.py:88-106, 121-141``."""
    v = np.asarray(values, dtype=np.float64)
    pts = v.shape[0]
    if mode == "midpoint":
        return np.column_stack([np.ones(pts), v]), dt, pts
    if mode in ("gauss2", "gauss4"):
        return gauss_table(v, dt, mode == "gauss4")
    c1, c2, c3 = v[0:pts - 1:2], v[1:pts:2], v[2:pts:2]
    if mode == "simpson":
        table = np.column_stack([np.ones(c1.shape[0]), (c1 + 4.0 * c2 + c3) / 6.0])
        return table, 2.0 * dt, c1.shape[0]
    n = v.shape[1]
    simpson = dt * (c1 + 4.0 * c2 + c3) / 3.0
    drift = (dt * dt / 3.0) * (c3 - c1)
    pairs = [(k, kp) for k in range(n) for kp in range(k + 1, n)]
    cross = np.empty((c1.shape[0], len(pairs)))
    for col, (k, kp) in enumerate(pairs):
        cross[:, col] = (dt * dt / 3.0) * (c1[:, k] * c3[:, kp] - c3[:, k] * c1[:, kp])
    coeffs = np.column_stack([simpson, drift, cross])
    scale = 2.0 * dt
    table = np.empty((coeffs.shape[0], 1 + coeffs.shape[1]))
    table[:, 0] = 1.0
    table[:, 1:] = coeffs / scale
    return table, scale, c1.shape[0]


def gauss_table(v: np.ndarray, dt: float, magnus: bool):
    """Gauss-Legendre modes (north-star extension; no reference to pin —
    "parity unpinned" for these rows, checked by convergence order instead):
    slice k = rows a = 2k, b = 2k + 1 sampled at the Gauss nodes of a slice
    of length h = 2 dt.  Omega = -i G with G = (h/2)(H(a) + H(b)) +
    (sqrt(3) h^2 / 12) i[H(a), H(b)] (4th-order Magnus, Blanes-Casas-Ros
    2000); expanded over [H0, Hk, i[H0,Hk], i[Hk,Hk']] at scale h the
    weights are (a + b)/2, (sqrt(3) dt / 6)(b - a) and
    (sqrt(3) dt / 6)(a_k b_k' - a_k' b_k).  gauss2 keeps the first column
    only (2nd order)."""
    a, b = v[0::2], v[1::2]
    count = a.shape[0]
    cols = [np.ones(count), 0.5 * (a + b)]
    if magnus:
        g = math.sqrt(3.0) * dt / 6.0
        n = v.shape[1]
        pairs = [(k, kp) for k in range(n) for kp in range(k + 1, n)]
        cross = np.empty((count, len(pairs)))
        for col, (k, kp) in enumerate(pairs):
            cross[:, col] = g * (a[:, k] * b[:, kp] - a[:, kp] * b[:, k])
        cols += [g * (b - a), cross]
    return np.column_stack(cols), 2.0 * dt, count


def spectral_bound(dt: float, mode: str, base_norms, dcomm_norms=(), ccomm_norms=()) -> float:
    """beta (``hamiltonian.py:156-162``, ``magnus.py:109-118``,
    step selection ``propagator.py:258-262``)."""
    if mode == "gauss4":  # |weights| <= 1, sqrt(3) dt / 3 at scale 2 dt
        return (2.0 * dt * sum(base_norms)
                + (2.0 * math.sqrt(3.0) * dt * dt / 3.0) * (sum(dcomm_norms) + sum(ccomm_norms)))
    if mode == "magnus":
        return (2.0 * dt * sum(base_norms)
                + (2.0 * dt * dt / 3.0) * sum(dcomm_norms)
                + (2.0 * dt * dt / 3.0) * sum(ccomm_norms))
    step = dt if mode == "midpoint" else 2.0 * dt
    return float(step) * sum(base_norms)


# --------------------------------------------------------------------------
# batched kernels (linalg.py:204-288, chebyshev.py:259-306, propagator.py:68-102)
# --------------------------------------------------------------------------

def expand(terms, table, scale, bits: int) -> np.ndarray:
    """G[k] = scale * sum_i table[k,i] terms[i] as two flattened GEMMs
    (``linalg.py:246-288``)."""
    cdt = complex_dtype(bits)
    d = terms[0].shape[0]
    pts = table.shape[0]
    flat = np.stack([np.asarray(t).reshape(d * d) for t in terms]).astype(cdt)
    tab = np.asarray(table, dtype=np.float64).astype(cdt)
    view = np.empty((pts, d * d), dtype=cdt)
    np.matmul(tab[:, :1], flat[:1], out=view)
    if len(terms) > 1:
        step = max(1, _GEMM_BLOCK_BYTES // (d * d * view.dtype.itemsize))
        buf = np.empty((min(step, pts), d * d), dtype=cdt)
        for lo in range(0, pts, step):
            hi = min(lo + step, pts)
            blk = buf[:hi - lo]
            np.matmul(tab[lo:hi, 1:], flat[1:], out=blk)
            view[lo:hi] += blk
    if scale != 1:
        view *= real_dtype(bits).type(scale)
    return view.reshape(pts, d, d)


def _gemm_acc(a, b, alpha, beta, c):
    """c = alpha a b + beta c, beta != 0, blocked (``linalg.py:225-232``)."""
    dt = c.dtype
    if beta != 1:
        c *= dt.type(beta)
    d = c.shape[-1]
    step = max(1, _GEMM_BLOCK_BYTES // (d * d * dt.itemsize))
    buf = np.empty((min(step, c.shape[0]), d, d), dtype=dt)
    for lo in range(0, c.shape[0], step):
        hi = min(lo + step, c.shape[0])
        blk = buf[:hi - lo]
        np.matmul(a[lo:hi], b[lo:hi], out=blk)
        if alpha != 1:
            blk *= dt.type(alpha)
        c[lo:hi] += blk


def expm_clenshaw(g: np.ndarray, plan: dict, bits: int) -> np.ndarray:
    """exp(-iG) per slice by the fused two-step Clenshaw descent
    (``chebyshev.py:259-306``): X = (2/span)(G - center I); for k = m, m-2,
    .., 1: D1 <- 2 X D0 - D1 + a_k I;  D0 <- 2 X D1 - (2 if k == 1 else 1) D0
    + (a_0 if k == 1 else a_{k-1}) I; result phase * D0."""
    cdt = complex_dtype(bits)
    n, d, _ = g.shape
    span = plan["beta"] - plan["alpha"]
    center = 0.5 * (plan["alpha"] + plan["beta"])
    if span == 0.0:
        x = np.zeros_like(g)
    else:
        x = g.copy()
        if center != 0.0:
            idx = np.arange(d)
            x[:, idx, idx] += cdt.type(-center)
        x *= real_dtype(bits).type(2.0 / span)
    a = plan["coeffs"].astype(cdt)
    d0 = np.zeros((n, d, d), dtype=cdt)
    d1 = np.zeros((n, d, d), dtype=cdt)
    idx = np.arange(d)
    for k in range(plan["m_max"], 0, -2):
        _gemm_acc(x, d0, 2.0, -1.0, d1)
        d1[:, idx, idx] += a[k]
        last = k == 1
        _gemm_acc(x, d1, 2.0, -2.0 if last else -1.0, d0)
        d0[:, idx, idx] += a[0] if last else a[k - 1]
    if plan["phase"] != 1.0:
        d0 *= cdt.type(plan["phase"])
    return d0


def reduce_pairwise(u: np.ndarray) -> np.ndarray:
    """Level-order fold, later slice on the left, odd carry copied forward
    (``propagator.py:68-102``)."""
    n = u.shape[0]
    if n == 0:
        return np.eye(u.shape[1], dtype=u.dtype)
    src = u
    while src.shape[0] > 1:
        pairs = src.shape[0] // 2
        nxt = np.empty((pairs + src.shape[0] % 2,) + src.shape[1:], dtype=src.dtype)
        np.matmul(src[1:2 * pairs:2], src[0:2 * pairs:2], out=nxt[:pairs])
        if src.shape[0] % 2:
            nxt[pairs] = src[-1]
        src = nxt
    return src[0].copy()


def reduce_sequential(u: np.ndarray) -> np.ndarray:
    """acc = U[k] @ acc (``propagator.py:303-307``)."""
    acc = u[0].copy()
    for k in range(1, u.shape[0]):
        acc = np.matmul(u[k], acc)
    return acc


def cumulative(u: np.ndarray) -> np.ndarray:
    """cum[k] = U[k] @ cum[k-1] (``propagator.py:326-330``)."""
    cum = np.empty_like(u)
    if u.shape[0]:
        cum[0] = u[0]
    for k in range(1, u.shape[0]):
        cum[k] = np.matmul(u[k], cum[k - 1])
    return cum


# --------------------------------------------------------------------------
# the equiprop pipeline (propagator.py:238-331)
# --------------------------------------------------------------------------

def slice_propagators(h0, hs, values, dt, *, mode="midpoint", bits=64, m_max=None):
    """(U batch, plan) — expand, bound, plan, chunked Clenshaw
    (``propagator.py:238-277``).  mode in {midpoint, simpson, magnus} (+ the
    gauss2 / gauss4 extensions)."""
    magnus = mode in ("magnus", "gauss4")
    terms, bn, dn, cn = effective_terms(h0, hs, magnus)
    table, scale, count = slice_table(values, dt, mode)
    g = expand(terms, table, scale, bits)
    beta = spectral_bound(dt, mode, bn, dn, cn)
    plan = make_plan(-beta, beta, bits, m_max)
    d = g.shape[1]
    chunk = max(1, _EXPM_CHUNK_BYTES // (d * d * complex_dtype(bits).itemsize))
    if count <= chunk:
        return expm_clenshaw(g, plan, bits), plan
    for lo in range(0, count, chunk):
        hi = min(lo + chunk, count)
        g[lo:hi] = expm_clenshaw(g[lo:hi], plan, bits)
    return g, plan


def _summary(plan):
    return {k: plan[k] for k in ("alpha", "beta", "m_max", "predicted_error")}


def equiprop(h0, hs, values, dt, *, mode="midpoint", bits=64, m_max=None,
             reduction="pairwise"):
    """(U_total, slice_count, plan summary) (``propagator.py:279-308``)."""
    values = np.asarray(values, dtype=np.float64)
    d = np.asarray(h0).shape[0]
    if values.shape[0] == 0:
        return np.eye(d, dtype=complex_dtype(bits)), 0, None
    u, plan = slice_propagators(h0, hs, values, dt, mode=mode, bits=bits, m_max=m_max)
    total = reduce_pairwise(u) if reduction == "pairwise" else reduce_sequential(u)
    return total, u.shape[0], _summary(plan)


def equiprop_all(h0, hs, values, dt, *, mode="midpoint", bits=64, m_max=None):
    """(cumulative stack, slice_count, plan summary) (``propagator.py:310-331``)."""
    values = np.asarray(values, dtype=np.float64)
    d = np.asarray(h0).shape[0]
    if values.shape[0] == 0:
        return np.zeros((0, d, d), dtype=complex_dtype(bits)), 0, None
    u, plan = slice_propagators(h0, hs, values, dt, mode=mode, bits=bits, m_max=m_max)
    return cumulative(u), u.shape[0], _summary(plan)


# --------------------------------------------------------------------------
# extended-precision analytic oracle for the driven qubit (studies.py:123-153)
# --------------------------------------------------------------------------

def midpoint_reference_ld(w0, w1, wrf, duration, steps, chunk=1 << 16):
    """Midpoint-sliced driven-qubit propagator from exact per-slice SU(2)
    rotations, evaluated in 80-bit long double with a pairwise fold
    (``studies.py:123-153`` recipe; SURVEY.md §8(c) extended oracle)."""
    L = np.longdouble
    if steps < 1:
        return np.eye(2, dtype=complex)
    dt = L(duration) / L(steps)
    vnorm = np.hypot(L(w1), L(w0))
    half = vnorm * dt / L(2)
    c, s = np.cos(half), np.sin(half)
    ax, az = L(w1) / vnorm, L(w0) / vnorm

    def mul(a, b):  # (re, im) pairs of (.., 2, 2) long double arrays
        ar, ai = a
        br, bi = b
        return (ar @ br - ai @ bi, ar @ bi + ai @ br)

    total = (np.eye(2, dtype=L), np.zeros((2, 2), dtype=L))
    for lo in range(0, steps, chunk):
        k = np.arange(lo, min(lo + chunk, steps), dtype=L)
        ph = L(wrf) * (k + L(0.5)) * dt
        cx, sy = ax * np.cos(ph), ax * np.sin(ph)
        m = k.size
        ur = np.zeros((m, 2, 2), dtype=L)
        ui = np.zeros((m, 2, 2), dtype=L)
        ur[:, 0, 0] = c
        ui[:, 0, 0] = -s * az
        ur[:, 1, 1] = c
        ui[:, 1, 1] = s * az
        # -i s (nx - i ny) = -s ny - i s nx ; -i s (nx + i ny) = s ny - i s nx
        ur[:, 0, 1] = -s * sy
        ui[:, 0, 1] = -s * cx
        ur[:, 1, 0] = s * sy
        ui[:, 1, 0] = -s * cx
        u = (ur, ui)
        while u[0].shape[0] > 1:
            p = u[0].shape[0] // 2
            nr, ni = mul((u[0][1:2 * p:2], u[1][1:2 * p:2]), (u[0][0:2 * p:2], u[1][0:2 * p:2]))
            if u[0].shape[0] % 2:
                nr = np.concatenate([nr, u[0][-1:]])
                ni = np.concatenate([ni, u[1][-1:]])
            u = (nr, ni)
        total = mul((u[0][0], u[1][0]), total)
    return (total[0].astype(np.float64) + 1j * total[1].astype(np.float64))
