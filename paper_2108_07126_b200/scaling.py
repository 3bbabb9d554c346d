"""Scaling and squaring past the series capability (north-star extension).

The reference refuses a step whose global spectral bound beta exceeds the
Chebyshev capability of the largest order (4.447 fp64 / 9.919 fp32,
``chebyshev.py:113-134``: ``StepTooLargeError``), and so does this package by
default.  A context created with ``scaling=True`` (or after
``ctx.set_scaling(True)``) propagates such steps instead:

1. per-slice norm bounds nu_k = scale * sum_i |w_{k,i}| ||T_i||_1 from the
   slice's own weights (the reference's bound, ``hamiltonian.py:156-162`` /
   ``magnus.py:109-118``, with the slice's samples in place of |c| <= 1);
2. per chunk of slices, the order m and squaring count s minimising
   (m + 1) + 2 s subject to max_k nu_k / 2^s <= capability(m) (a squaring
   costs a GEMM and doubles the propagated rounding, so it counts twice) — the same
   Chebyshev plan machinery at the reduced bound beta' = max nu / 2^s;
3. on the device: the exponents G_k / 2^s (``sp_expand_batch_device``), their
   plan polynomials (``sp_expm_batch_device``), s batched squarings
   U <- U U (``sp_gemm_batched_device``), the chunk's ordered product
   (``sp_product_device``, pairwise or sequential as requested), chunks
   multiplied in time order.

It is the materialised path (exponents and propagators of one chunk in HBM,
256 MiB per chunk) — an extension for steps the fused lane kernels cannot
take, not the hot path: whenever beta is within the capability, ``equiprop``
runs the fused kernels exactly as without scaling.  Parity is gated against
an independent eigendecomposition oracle (``tests/test_scaling_gpu.py``).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from ._native import check, lib
from .chebyshev import ORDER_GRID, make_plan, norm_capability
from .hamiltonian import Quadrature, check_pair, simpson_triplets
from .linalg import Precision, one_norm
from .magnus import magnus_coefficients

CHUNK_BYTES = 256 << 20


def slice_table(ctx, amps) -> tuple[np.ndarray, float]:
    """(count, T) weight table (column 0 = the drift's unit weight) and the
    exponent scale of the loaded mode: midpoint [1, c_k] at dt
    (``hamiltonian.py:199-201``); Simpson [1, (c1 + 4 c2 + c3)/6] at 2 dt
    (``:202-205``); Magnus [1, table / (2 dt)] at 2 dt (``magnus.py:121-141``)."""
    if ctx._quadrature is Quadrature.GAUSS:
        from .magnus import gauss_table
        return gauss_table(amps, ctx._magnus)
    if ctx._magnus:
        coeffs = magnus_coefficients(amps)
        scale = 2.0 * amps.dt
        return np.column_stack([np.ones(coeffs.shape[0]), coeffs / scale]), scale
    if ctx._quadrature is Quadrature.MIDPOINT:
        return np.column_stack([np.ones(amps.pts), amps.values]), amps.dt
    c1, c2, c3 = simpson_triplets(amps.values)
    return (np.column_stack([np.ones(c1.shape[0]), (c1 + 4.0 * c2 + c3) / 6.0]),
            2.0 * amps.dt)


def slice_bounds(table: np.ndarray, scale: float, norms: np.ndarray) -> np.ndarray:
    """Per-slice 1-norm bound of the exponent G_k."""
    return scale * (np.abs(table) @ norms)


def schedule(nu: float, precision: Precision, m_max: int | None = None) -> tuple[int, int]:
    """(m, s) minimising (m + 1) GEMMs + 2 s (squarings) with nu / 2^s within
    the order-m capability; ties go to fewer squarings."""
    best = None
    for m in ([m_max] if m_max else ORDER_GRID):
        cap = norm_capability(m, precision)
        s = 0 if nu <= cap else int(math.ceil(math.log2(nu / cap)))
        while nu / 2.0 ** s > cap:  # guard the log rounding
            s += 1
        key = (m + 1 + 2 * s, s)
        if best is None or key < best[0]:
            best = (key, m, s)
    return best[1], best[2]


def equiprop_scaled(ctx, amps, reduction: str):
    """Total propagator of a step past the capability (module docstring)."""
    import torch

    from .propagator import PropagatorResult

    check_pair(ctx._system, amps)  # |c| <= 1 with the reference's message, on the host
    precision = ctx.precision
    bits = precision.bits
    terms = ctx._effective.terms() if ctx._magnus else ctx._system.terms()
    norms = np.array([one_norm(t) for t in terms])
    table, scale = slice_table(ctx, amps)
    count = table.shape[0]
    d = ctx._system.dim
    dd = d * d
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev)
    sp_stream = ctypes.c_void_p(stream.cuda_stream)
    cdt = torch.complex64 if bits == 32 else torch.complex128
    d_terms = torch.from_numpy(np.ascontiguousarray(np.stack(terms), dtype=np.complex128)
                               ).to(dev)
    nu = slice_bounds(table, scale, norms)
    chunk = max(1, min(count, CHUNK_BYTES // (dd * 16)))
    total = torch.eye(d, dtype=torch.complex128, device=dev)
    # the context writes products in its working dtype (complex64 for fp32)
    prod = torch.empty((d, d), dtype=cdt, device=dev)
    nxt = torch.empty((d, d), dtype=torch.complex128, device=dev)
    used_m, used_s = None, 0
    for lo in range(0, count, chunk):
        c = min(chunk, count - lo)
        nu_max = float(nu[lo:lo + c].max())
        m, s = schedule(nu_max, precision, ctx.m_max)
        beta = nu_max / 2.0 ** s
        plan = make_plan(-beta, beta, precision, m_max=m)
        used_m, used_s = m if used_m is None else max(used_m, m), max(used_s, s)
        d_coef = torch.from_numpy(np.ascontiguousarray(table[lo:lo + c])).to(dev)
        g = torch.empty((c, d, d), dtype=cdt, device=dev)
        check(lib.sp_expand_batch_device(bits, d, len(terms), ctypes.c_void_p(d_terms.data_ptr()),
                                         c, ctypes.c_void_p(d_coef.data_ptr()),
                                         float(scale / 2.0 ** s), ctypes.c_void_p(g.data_ptr()),
                                         sp_stream))
        u = torch.empty_like(g)
        nbytes = lib.sp_expm_batch_scratch_bytes(bits, d, c)
        scratch = torch.empty(max(1, nbytes), dtype=torch.uint8, device=dev)
        native = plan.to_native()
        check(lib.sp_expm_batch_device(bits, d, c, ctypes.c_void_p(g.data_ptr()), dd,
                                       ctypes.byref(native), ctypes.c_void_p(u.data_ptr()), dd,
                                       ctypes.c_void_p(scratch.data_ptr()), sp_stream))
        for _ in range(s):  # U <- U U (A and B alias; C is the other buffer)
            check(lib.sp_gemm_batched_device(bits, d, c, ctypes.c_void_p(u.data_ptr()), dd,
                                             ctypes.c_void_p(u.data_ptr()), dd, None, None,
                                             None, ctypes.c_void_p(g.data_ptr()), dd,
                                             sp_stream))
            u, g = g, u
        mats = u if bits == 64 else u.to(torch.complex128)
        ctx.product_device_ptr(c, mats.data_ptr(), prod.data_ptr(), stream=stream.cuda_stream,
                               reduction=reduction)
        # total <- (chunk product) total
        p128 = prod if bits == 64 else prod.to(torch.complex128)
        check(lib.sp_gemm_batched_device(64, d, 1, ctypes.c_void_p(p128.data_ptr()), 0,
                                         ctypes.c_void_p(total.data_ptr()), 0, None, None, None,
                                         ctypes.c_void_p(nxt.data_ptr()), 0, sp_stream))
        total, nxt = nxt, total
    stream.synchronize()
    u_host = total.cpu().numpy()
    if bits == 32:
        u_host = u_host.astype(np.complex64)
    beta = ctx.bound(amps.dt)
    summary = {"alpha": -beta, "beta": beta, "m_max": used_m,
               "predicted_error": None, "squarings": used_s,
               "max_slice_bound": float(nu.max())}
    return PropagatorResult(u=u_host, slice_count=count, plan=summary)
