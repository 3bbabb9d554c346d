"""Chebyshev plan for exp(-iG): order selection and series coefficients.

Same contract as the reference ``sliceprop/chebyshev.py:1-218``; the
arithmetic runs in the C++ host plan of the native library
(``csrc/plan.cpp``: 80-bit Miller recurrence for J_k, libm exp/pow for the
error estimate), bit-for-bit equal to the reference (tests/test_plan.py).
The series itself is evaluated on the GPU inside the lane kernels.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from ._native import lib
from .errors import ConfigError, DomainError, StepTooLargeError, raise_for
from .linalg import Precision

__all__ = [
    "ORDER_GRID",
    "bessel_j",
    "chebyshev_error",
    "select_m_max",
    "norm_capability",
    "ChebyshevPlan",
    "make_plan",
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


