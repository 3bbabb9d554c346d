"""B200 backend for the reference package — the module a sliceprop maintainer
adds as ``sliceprop/b200.py``.

It binds the C ABI of ``include/sliceprop_b200.h`` (``libsliceprop_b200.so``;
path from ``SLICEPROP_B200_LIB``) with ctypes, the reference's natural FFI,
and routes the propagation hot path of ``IntegratorContext`` through it:

* ``create(backend="b200")`` attaches a ``B200Backend`` (one native context
  per Python context; ``devices=[...]`` spreads one propagation over several
  GPUs of this process);
* ``set_hamiltonian`` loads the expansion terms once (drift + controls, or
  the Magnus effective system of ``build_effective_system``);
* ``equiprop`` / ``equiprop_all`` keep the reference's validation order
  (reduction token -> state -> type -> empty table -> sampling parity ->
  control count and |c| <= 1 -> bound and plan / StepTooLargeError,
  ``propagator.py:238-331``) and then make ONE library call instead of
  ``_slice_propagators`` + ``reduce_pairwise``.

Everything else in ``sliceprop`` is unchanged; contexts created without the
token keep the CPU backend.  ``install()`` applies the three hooks to the
package's ``propagator`` module (the patch a maintainer would make by hand).
"""

import ctypes
import os

import numpy as np

from . import propagator as _prop
from .errors import (AmplitudeBoundError, ConfigError, DomainError, HermiticityError,
                     IntegratorError, SamplingParityError, ShapeError, StateMachineError,
                     StepTooLargeError)
from .hamiltonian import ControlAmplitudes, Quadrature, _check_pair, spectral_bound
from .magnus import magnus_spectral_bound

_P = ctypes.c_void_p
_lib = ctypes.CDLL(os.environ.get("SLICEPROP_B200_LIB", "libsliceprop_b200.so"))


class _Plan(ctypes.Structure):  # sp_plan
    _fields_ = [("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("m_max", ctypes.c_int), ("coeffs", ctypes.c_double * 52),
                ("phase", ctypes.c_double * 2), ("predicted_error", ctypes.c_double),
                ("capability", ctypes.c_double), ("norm_bound", ctypes.c_double)]


_lib.sp_create.argtypes = [ctypes.POINTER(_P), ctypes.c_int, ctypes.c_int,
                           ctypes.POINTER(ctypes.c_int)]
_lib.sp_free.argtypes = [_P]
_lib.sp_set_hamiltonian.argtypes = [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, _P]
_lib.sp_equiprop.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                             ctypes.POINTER(_Plan), ctypes.c_int, _P]
_lib.sp_equiprop_all.argtypes = [_P, _P, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                 ctypes.POINTER(_Plan), _P]
_lib.sp_last_error.argtypes = [_P]
_lib.sp_last_error.restype = ctypes.c_char_p
_CODES = {1: ShapeError, 2: HermiticityError, 3: AmplitudeBoundError, 4: SamplingParityError,
          5: StepTooLargeError, 6: StateMachineError, 8: DomainError, 9: ConfigError}


def _check(rc, handle):
    if rc:
        msg = _lib.sp_last_error(handle)
        raise _CODES.get(rc, IntegratorError)(msg.decode() if msg else f"error {rc}")


class B200Backend:
    """One native propagation context (``sp_create``) on one or more GPUs."""

    name = "b200"

    def __init__(self, precision, devices=(0,)):
        self.bits = 32 if precision.value == "fp32" else 64
        ids = (ctypes.c_int * len(devices))(*devices)
        self._h = _P()
        _check(_lib.sp_create(ctypes.byref(self._h), self.bits, len(devices), ids), None)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.sp_free(self._h)
            self._h = _P()

    def load(self, terms, n_controls, mode):  # mode 0 midpoint, 1 simpson, 2 magnus
        t = np.ascontiguousarray(np.stack(terms), dtype=np.complex128)
        _check(_lib.sp_set_hamiltonian(self._h, t.shape[1], n_controls, t.shape[0], mode,
                                       t.ctypes.data_as(_P)), self._h)

    @staticmethod
    def _plan(plan):
        p = _Plan(alpha=plan.alpha, beta=plan.beta, m_max=plan.m_max)
        for k, a in enumerate(plan.coeffs):
            p.coeffs[2 * k], p.coeffs[2 * k + 1] = a.real, a.imag
        p.phase[0], p.phase[1] = plan.phase.real, plan.phase.imag
        return p

    def equiprop(self, amps, plan, reduction, out):
        _check(_lib.sp_equiprop(self._h, amps.values.ctypes.data_as(_P), amps.pts,
                                amps.n_controls, amps.dt, ctypes.byref(self._plan(plan)),
                                0 if reduction == "pairwise" else 1,
                                out.ctypes.data_as(_P)), self._h)
        return out

    def equiprop_all(self, amps, plan, out):
        _check(_lib.sp_equiprop_all(self._h, amps.values.ctypes.data_as(_P), amps.pts,
                                    amps.n_controls, amps.dt, ctypes.byref(self._plan(plan)),
                                    out.ctypes.data_as(_P)), self._h)
        return out


def _prepare(ctx, amps):
    """The reference's checks of _slice_propagators (propagator.py:238-266)."""
    if ctx._quadrature is Quadrature.SIMPSON:
        if amps.pts < 3 or amps.pts % 2 == 0:
            raise SamplingParityError(
                f"three-point quadrature needs an odd number of samples >= 3, got {amps.pts}")
        count = (amps.pts - 1) // 2
    else:
        count = amps.pts
    _check_pair(ctx._system, amps)
    if ctx._magnus:
        bound = magnus_spectral_bound(ctx._effective, amps)
    else:
        step = amps.dt if ctx._quadrature is Quadrature.MIDPOINT else 2.0 * amps.dt
        bound = spectral_bound(ctx._system, step)
    plan = _prop.make_plan(-bound, bound, ctx.precision, m_max=ctx.m_max)
    return count, plan


def _state_checks(ctx, amps):
    ctx._require_open()
    if ctx._state != _prop._LOADED:
        raise StateMachineError("no Hamiltonian loaded; call set_hamiltonian first")
    if not isinstance(amps, ControlAmplitudes):
        raise ShapeError(f"expected ControlAmplitudes, got {type(amps).__name__}")


def install(default=False, devices=(0,)):
    """Hook the backend into ``sliceprop.propagator``.  ``default=True`` makes
    ``create()`` without a backend argument use the B200 (test harnesses)."""
    if getattr(_prop, "_b200_installed", False):
        return
    orig_create = _prop.create
    orig_set = _prop.IntegratorContext.set_hamiltonian
    orig_eq = _prop.IntegratorContext.equiprop
    orig_all = _prop.IntegratorContext.equiprop_all

    def create(precision="fp64", m_max=None, checked=False, backend=None):
        if (backend is None and default) or (isinstance(backend, str)
                                             and backend.lower() == "b200"):
            ctx = orig_create(precision, m_max, checked)
            ctx.backend = B200Backend(ctx.precision, devices)
            return ctx
        return orig_create(precision, m_max, checked, backend)

    def set_hamiltonian(self, system, magnus=False, quadrature=None):
        orig_set(self, system, magnus, quadrature)
        if isinstance(self.backend, B200Backend):
            terms = self._effective.terms() if self._magnus else system.terms()
            mode = 2 if self._magnus else (0 if self._quadrature is Quadrature.MIDPOINT else 1)
            self.backend.load(terms, system.n_controls, mode)

    def equiprop(self, amps, reduction="pairwise"):
        if not isinstance(self.backend, B200Backend):
            return orig_eq(self, amps, reduction)
        if reduction not in ("pairwise", "sequential"):
            raise ConfigError(f"unknown reduction {reduction!r}; expected pairwise or sequential")
        _state_checks(self, amps)
        d = self._system.dim
        if amps.pts == 0:
            return _prop.PropagatorResult(u=np.eye(d, dtype=self.precision.complex_dtype),
                                          slice_count=0, plan=None)
        count, plan = _prepare(self, amps)
        out = np.empty((d, d), dtype=self.precision.complex_dtype)
        self.backend.equiprop(amps, plan, reduction, out)
        return _prop.PropagatorResult(u=out, slice_count=count, plan=plan.summary())

    def equiprop_all(self, amps):
        if not isinstance(self.backend, B200Backend):
            return orig_all(self, amps)
        _state_checks(self, amps)
        d = self._system.dim
        cdt = self.precision.complex_dtype
        if amps.pts == 0:
            return _prop.CumulativeResult(u_all=np.zeros((0, d, d), dtype=cdt), slice_count=0,
                                          plan=None)
        count, plan = _prepare(self, amps)
        out = np.empty((count, d, d), dtype=cdt)
        self.backend.equiprop_all(amps, plan, out)
        return _prop.CumulativeResult(u_all=out, slice_count=count, plan=plan.summary())

    _prop.create = create
    _prop.IntegratorContext.set_hamiltonian = set_hamiltonian
    _prop.IntegratorContext.equiprop = equiprop
    _prop.IntegratorContext.equiprop_all = equiprop_all
    import sys
    pkg = sys.modules[__name__.rsplit(".", 1)[0]]
    pkg.create = create
    _prop._b200_installed = True
