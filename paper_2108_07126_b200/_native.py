"""ctypes binding of the sm_100a C-ABI library ``libsliceprop_b200.so``.

The library is built in-tree by ``paper_2108_07126_b200/build.py`` (called
from ``__graft_entry__.build()``).  There is no fallback: if the shared
object is missing, importing the package raises immediately, and any
propagation on a machine without a B200 fails with ``InternalError``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import raise_for

__all__ = ["lib", "SpPlan", "LIB_PATH", "HEADER_SYMBOLS", "check", "MODE", "REDUCTION"]

# SLICEPROP_B200_LIB selects an instrumented build of the same sources (tools/)
LIB_PATH = os.environ.get("SLICEPROP_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libsliceprop_b200.so")

MODE = {"midpoint": 0, "simpson": 1, "magnus": 2, "gauss2": 3, "gauss4": 4}
REDUCTION = {"pairwise": 0, "sequential": 1}
MAX_ORDER = 25


class SpPlan(ctypes.Structure):
    """Mirror of ``sp_plan`` (include/sliceprop_b200.h)."""

    _fields_ = [
        ("alpha", ctypes.c_double),
        ("beta", ctypes.c_double),
        ("m_max", ctypes.c_int),
        ("coeffs", ctypes.c_double * (2 * (MAX_ORDER + 1))),
        ("phase", ctypes.c_double * 2),
        ("predicted_error", ctypes.c_double),
        ("capability", ctypes.c_double),
        ("norm_bound", ctypes.c_double),
    ]


# every exported symbol of include/sliceprop_b200.h with its signature
_c = ctypes
_P = _c.c_void_p
HEADER_SYMBOLS = {
    "sp_version": (_c.c_char_p, []),
    "sp_bessel_j": (_c.c_int, [_c.c_int, _c.c_double, _c.POINTER(_c.c_double)]),
    "sp_chebyshev_error": (_c.c_double, [_c.c_int, _c.c_double]),
    "sp_select_m_max": (_c.c_int, [_c.c_double, _c.c_int, _c.POINTER(_c.c_int),
                                   _c.POINTER(_c.c_double)]),
    "sp_norm_capability": (_c.c_int, [_c.c_int, _c.c_int, _c.POINTER(_c.c_double)]),
    "sp_make_plan": (_c.c_int, [_c.c_double, _c.c_double, _c.c_int, _c.c_int,
                                _c.POINTER(SpPlan)]),
    "sp_create": (_c.c_int, [_c.POINTER(_P), _c.c_int, _c.c_int, _c.POINTER(_c.c_int)]),
    "sp_free": (_c.c_int, [_P]),
    "sp_last_error": (_c.c_char_p, [_P]),
    "sp_set_hamiltonian": (_c.c_int, [_P, _c.c_int, _c.c_int, _c.c_int, _c.c_int, _P]),
    "sp_equiprop": (_c.c_int, [_P, _P, _c.c_int64, _c.c_int, _c.c_double,
                               _c.POINTER(SpPlan), _c.c_int, _P]),
    "sp_equiprop_device": (_c.c_int, [_P, _P, _c.c_int64, _c.c_int, _c.c_double,
                                      _c.POINTER(SpPlan), _c.c_int, _P, _P]),
    "sp_equiprop_all": (_c.c_int, [_P, _P, _c.c_int64, _c.c_int, _c.c_double,
                                   _c.POINTER(SpPlan), _P]),
    "sp_equiprop_all_device": (_c.c_int, [_P, _P, _c.c_int64, _c.c_int, _c.c_double,
                                          _c.POINTER(SpPlan), _P, _P]),
    "sp_product_device": (_c.c_int, [_P, _c.c_int, _P, _c.c_int, _P, _P]),
    "sp_slice_count": (_c.c_int, [_P, _c.c_int64, _c.POINTER(_c.c_int64)]),
    "sp_amplitude_violation": (_c.c_int, [_P, _c.POINTER(_c.c_int64)]),
    "sp_set_algorithm": (_c.c_int, [_P, _c.c_int]),
    "sp_last_algorithm": (_c.c_int, [_P, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "sp_expand_batch_device": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int, _P, _c.c_int64, _P,
                                          _c.c_double, _P, _P]),
    "sp_expm_batch_scratch_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _c.c_int64]),
    "sp_expm_batch_device": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int64, _P, _c.c_int64,
                                        _c.POINTER(SpPlan), _P, _c.c_int64, _P, _P]),
    "sp_gemm_batched_device": (_c.c_int, [_c.c_int, _c.c_int, _c.c_int64, _P, _c.c_int64, _P,
                                          _c.c_int64, _P, _P, _P, _P, _c.c_int64, _P]),
    "sp_apply_batch_scratch_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _c.c_int64, _c.c_int]),
    "sp_apply_batch_device": (_c.c_int, [_c.c_int, _c.c_int, _P, _c.c_int64, _c.c_int, _P, _P,
                                         _P, _P]),
    "sp_qubit_midpoint_reference": (_c.c_int, [_P, _c.c_double, _c.c_double, _c.c_double,
                                               _c.c_double, _c.c_int64, _P]),
    "sp_last_lanes": (_c.c_int, [_P, _c.POINTER(_c.c_int)]),
    "sp_set_profiling": (_c.c_int, [_P, _c.c_int]),
    "sp_last_timing": (_c.c_int, [_P, _c.POINTER(_c.c_double), _c.POINTER(_c.c_int),
                                  _c.POINTER(_c.c_double), _c.c_char_p, _c.c_int]),
    "sp_device_count": (_c.c_int, [_c.POINTER(_c.c_int)]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__ as g; g.build()').  There is no CPU "
            "fallback for the propagation path.")
    handle = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in HEADER_SYMBOLS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


lib = _load()


def check(rc: int, ctx=None, **extra) -> None:
    """Raise the reference exception class for a non-zero C-ABI code."""
    if rc:
        msg = lib.sp_last_error(ctx)
        raise_for(rc, msg.decode() if msg else f"error code {rc}", **extra)
