"""Chebyshev plan for exp(-iG): order selection and series coefficients.

Same contract as the reference ``sliceprop/chebyshev.py:1-218``; the
arithmetic runs in the C++ host plan of the native library
(``csrc/plan.cpp``: 80-bit Miller recurrence for J_k, libm exp/pow for the
error estimate), bit-for-bit equal to the reference (tests/test_plan.py).
The series itself is evaluated on the GPU: inside the lane kernels for
equiprop, and by the batch kernels (``csrc/kernels_batch.cuh``) for the
standalone ``expm_batch`` over a user's own exponent batch
(``chebyshev.py:221-306``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import lib
from .errors import (ConfigError, DomainError, HermiticityError, ShapeError, StepTooLargeError,
                     raise_for)
from .linalg import DeviceBackend, MatrixBatch, Precision, default_backend

__all__ = [
    "ORDER_GRID",
    "bessel_j",
    "chebyshev_error",
    "select_m_max",
    "norm_capability",
    "ChebyshevPlan",
    "make_plan",
    "Workspace",
    "expm_batch",
]

# odd truncation orders the selector may choose from (chebyshev.py:50-51)
ORDER_GRID = tuple(range(3, 26, 2))


def _last_error() -> str:
    msg = lib.sp_last_error(None)
    return msg.decode() if msg else ""


def bessel_j(k: int, x: float) -> float:
    """Bessel function J_k(x), 0 <= k <= 64, 0 <= x <= 64 (``chebyshev.py:61-104``)."""
    if not isinstance(k, (int, np.integer)) or isinstance(k, bool):
        raise DomainError(f"order must be an integer, got {k!r}")
    x = float(x)
    if not (0 <= int(k) <= 64):
        raise DomainError(f"order {k} outside supported range 0..64")
    if not 0.0 <= x <= 64.0:
        raise DomainError(f"argument {x} outside supported range 0..64.0")
    out = ctypes.c_double()
    rc = lib.sp_bessel_j(int(k), x, ctypes.byref(out))
    if rc:
        raise_for(rc, _last_error())
    return out.value


def chebyshev_error(m: int, span: float) -> float:
    """Truncation error estimate 4 (e^{1-s^2} s)^{m+1}, s = span/(4m+4)."""
    return float(lib.sp_chebyshev_error(int(m), float(span)))


def norm_capability(m: int, precision) -> float:
    """Largest exponent norm g with chebyshev_error(m, 2g) at the precision target."""
    precision = Precision.parse(precision)
    if m not in ORDER_GRID:
        raise ConfigError(f"order {m} not in the supported grid {ORDER_GRID}")
    out = ctypes.c_double()
    rc = lib.sp_norm_capability(int(m), precision.bits, ctypes.byref(out))
    if rc:
        raise_for(rc, _last_error())
    return out.value


def select_m_max(norm_bound: float, precision) -> int:
    """Smallest odd order in 3..25 reaching the precision target (``:113-134``)."""
    precision = Precision.parse(precision)
    norm_bound = float(norm_bound)
    if norm_bound < 0:
        raise DomainError(f"norm bound must be >= 0, got {norm_bound}")
    m = ctypes.c_int()
    cap = ctypes.c_double()
    rc = lib.sp_select_m_max(norm_bound, precision.bits, ctypes.byref(m), ctypes.byref(cap))
    if rc:
        raise_for(rc, _last_error(), norm_bound=norm_bound, capability=cap.value)
    return m.value


@dataclass(frozen=True)
class ChebyshevPlan:
    """Immutable description of one truncated-series evaluation
    (``chebyshev.py:155-182``)."""

    alpha: float
    beta: float
    m_max: int
    coeffs: np.ndarray
    phase: complex
    precision: Precision
    predicted_error: float

    @property
    def span(self) -> float:
        return self.beta - self.alpha

    def summary(self) -> dict:
        return {
            "alpha": self.alpha,
            "beta": self.beta,
            "m_max": self.m_max,
            "predicted_error": self.predicted_error,
        }

    def to_native(self) -> _native.SpPlan:
        p = _native.SpPlan()
        p.alpha = self.alpha
        p.beta = self.beta
        p.m_max = self.m_max
        for k, a in enumerate(self.coeffs):
            p.coeffs[2 * k] = a.real
            p.coeffs[2 * k + 1] = a.imag
        p.phase[0] = self.phase.real
        p.phase[1] = self.phase.imag
        p.predicted_error = self.predicted_error
        return p


def make_plan(alpha: float, beta: float, precision, m_max: int | None = None) -> ChebyshevPlan:
    """Evaluation plan for spectra inside [alpha, beta] (``chebyshev.py:185-218``)."""
    precision = Precision.parse(precision)
    alpha, beta = float(alpha), float(beta)
    if m_max is not None and m_max not in ORDER_GRID:
        raise ConfigError(
            f"m_max override {m_max} not an odd integer in {ORDER_GRID[0]}..{ORDER_GRID[-1]}")
    p = _native.SpPlan()
    rc = lib.sp_make_plan(alpha, beta, precision.bits, int(m_max or 0), ctypes.byref(p))
    if rc:
        raise_for(rc, _last_error(), norm_bound=p.norm_bound, capability=p.capability)
    m = p.m_max
    coeffs = np.array([complex(p.coeffs[2 * k], p.coeffs[2 * k + 1]) for k in range(m + 1)],
                      dtype=np.complex128)
    phase = complex(p.phase[0], p.phase[1])
    if alpha + beta == 0.0:
        phase = 1.0 + 0.0j
    return ChebyshevPlan(alpha=alpha, beta=beta, m_max=m, coeffs=coeffs, phase=phase,
                         precision=precision, predicted_error=p.predicted_error)




class Workspace:
    """Scratch of ``expm_batch`` (``chebyshev.py:221-246``): three host
    batches X, D0, D1 sized like G, bound to one dimension and precision,
    capacity growing monotonically; the result of ``expm_batch`` is a view of
    D0 valid until the next call on the same workspace.  The device-side
    staging (input, output and, for d > 64, the X / D1 / D0 scratch of the
    multi-launch path) is owned here too and grows the same way, so
    back-to-back evaluations do not reallocate on either side."""

    def __init__(self, dim: int, precision):
        if dim < 1:
            raise ShapeError(f"dim must be >= 1, got {dim}")
        self.dim = int(dim)
        self.precision = Precision.parse(precision)
        self.capacity = 0
        self._x = self._d0 = self._d1 = None
        self._dev = {}

    def ensure(self, count: int):
        """Views of the three scratch batches with exactly ``count`` slices."""
        if self._x is None or count > self.capacity:
            self._x = MatrixBatch.zeros(self.dim, count, self.precision)
            self._d0 = MatrixBatch.zeros(self.dim, count, self.precision)
            self._d1 = MatrixBatch.zeros(self.dim, count, self.precision)
            self.capacity = count
        return (self._x.subview(0, count), self._d0.subview(0, count),
                self._d1.subview(0, count))

    def device_buffer(self, name: str, nbytes: int, device):
        """Monotone device byte buffer ``name`` of at least ``nbytes``."""
        import torch
        buf = self._dev.get(name)
        if buf is None or buf.numel() < nbytes or buf.device != device:
            buf = torch.empty(max(16, nbytes), dtype=torch.uint8, device=device)
            self._dev[name] = buf
        return buf


def _check_hermitian(g: MatrixBatch) -> None:
    """checked=True validation (``chebyshev.py:249-256``), host-side."""
    gv = g.matrices()
    asym = np.abs(gv - gv.conj().transpose(0, 2, 1)).max() if g.count else 0.0
    scale = np.abs(gv).max() if g.count else 0.0
    tol = 100.0 * g.precision.roundoff * max(1.0, scale * g.dim)
    if asym > tol:
        raise HermiticityError(f"exponent batch asymmetry {asym:.3g} exceeds tolerance {tol:.3g}")


def expm_batch(g: MatrixBatch, plan: ChebyshevPlan, workspace: Workspace,
               backend: DeviceBackend | None = None, checked: bool = False) -> MatrixBatch:
    """U[k] = exp(-i G[k]) for every matrix of the batch, on the B200
    (``chebyshev.py:259-306``): the plan's Chebyshev polynomial evaluated by
    the reference's Clenshaw recurrence, X = (2/span)(G - center I), in the
    batch's working precision (complex64 batches in FP32 arithmetic).
    d <= 64: one fused kernel keeps X and the iterates on chip; d > 64:
    m + 1 batched GEMM launches.  The returned batch aliases the workspace."""
    import torch

    from ._native import check, lib
    if backend is not None and not isinstance(backend, DeviceBackend):
        raise ConfigError(f"expm_batch runs on the B200 DeviceBackend, got {backend!r}")
    backend = backend or default_backend()
    if g.precision is not plan.precision:
        raise ShapeError(f"batch precision {g.precision.value} does not match plan "
                         f"{plan.precision.value}")
    if workspace.dim != g.dim or workspace.precision is not g.precision:
        raise ShapeError("workspace dimension or precision does not match the batch")
    if checked:
        _check_hermitian(g)
    x, d0, d1 = workspace.ensure(g.count)
    if g.count == 0:
        return d0
    dev = backend.torch_device()
    prec = g.precision
    isz = prec.complex_dtype.itemsize
    n, d = g.count, g.dim
    d_g = workspace.device_buffer("g", n * d * d * isz, dev)
    d_g[:n * d * d * isz].copy_(torch.from_numpy(
        np.ascontiguousarray(g.matrices()).reshape(-1).view(np.uint8)))
    d_u = workspace.device_buffer("u", n * d * d * isz, dev)
    scratch_bytes = int(lib.sp_expm_batch_scratch_bytes(prec.bits, d, n))
    d_s = workspace.device_buffer("scratch", scratch_bytes, dev) if scratch_bytes else None
    native = plan.to_native()
    stream = backend.stream()
    check(lib.sp_expm_batch_device(prec.bits, d, n, ctypes.c_void_p(d_g.data_ptr()), d * d,
                                   ctypes.byref(native), ctypes.c_void_p(d_u.data_ptr()), d * d,
                                   ctypes.c_void_p(d_s.data_ptr() if d_s is not None else 0),
                                   ctypes.c_void_p(stream)))
    # batched products executed: the fused kernel skips the reference's first
    # multiply-by-zero, the d > 64 path runs all m + 1
    backend.gemm_calls += plan.m_max + (1 if d > 64 else 0)
    d0.matrices()[:] = d_u[:n * d * d * isz].cpu().numpy().view(prec.complex_dtype).reshape(n, d, d)
    return d0
