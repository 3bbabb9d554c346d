"""Equidistant propagation on the B200: the ``create`` / ``IntegratorContext``
drop-in for the reference ``sliceprop/propagator.py``.

The host keeps the reference's contract — lifecycle created -> loaded ->
closed (``propagator.py:121-216``), mode resolution (``:175-201``), the
order of validation (``:238-308``), the global spectral bound and the
Chebyshev plan (``:258-263``) — and hands the propagation itself to the
sm_100a library through one C-ABI call (``sp_equiprop`` /
``sp_equiprop_all``).  There is no CPU path: on a machine without a B200 the
call raises ``InternalError``.

Result ordering: U = U[n-1] ... U[0] (later slice on the left).  The device
multiplies slices inside contiguous lanes and then combines the lane
products in time order, pairwise (tree) or sequentially (left fold) — the
same products as the reference in a different association, so results agree
to rounding (tests/test_parity_gpu.py states the tolerances).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from ._native import MODE, REDUCTION, check, lib
from .chebyshev import ORDER_GRID, ChebyshevPlan, make_plan
from .errors import (AmplitudeBoundError, ConfigError, HermiticityError, SamplingParityError,
                     ShapeError, StepTooLargeError,
                     StateMachineError)
from .hamiltonian import (ControlAmplitudes, ControlSystem, Quadrature, check_pair,
                          simpson_triplets, spectral_bound)
from .linalg import DeviceBackend, Precision
from .magnus import EffectiveSystem, build_effective_system, magnus_bound

__all__ = [
    "IntegratorContext",
    "PropagatorResult",
    "CumulativeResult",
    "create",
    "apply",
    "apply_batch",
]

_CREATED, _LOADED, _CLOSED = "created", "loaded", "closed"

BACKEND_NAME = "b200"
_BACKEND_TOKENS = ("b200", "cuda", "gpu", "sm_100a")


@dataclass(frozen=True)
class PropagatorResult:
    """Total propagator plus bookkeeping (``propagator.py:31-41``)."""

    u: np.ndarray
    slice_count: int
    plan: dict | None

    @property
    def dim(self) -> int:
        return self.u.shape[0]


@dataclass(frozen=True)
class CumulativeResult:
    """Running products U(t_k <- 0) at every slice boundary
    (``propagator.py:44-65``).  ``u_all[-1]`` equals the sequential-reduction
    total of the same call bit for bit."""

    u_all: np.ndarray
    slice_count: int
    plan: dict | None

    @property
    def dim(self) -> int:
        return self.u_all.shape[1]

    @property
    def final(self) -> np.ndarray:
        if self.slice_count == 0:
            return np.eye(self.dim, dtype=self.u_all.dtype)
        return self.u_all[-1]


def apply(u, state) -> np.ndarray:
    """Propagate a state vector (U psi) or a density matrix (U rho U^+)
    (``propagator.py:105-118``) on the device (``sp_apply_batch_device``);
    same shapes, dtype and errors as the reference."""
    m = u.u if isinstance(u, PropagatorResult) else np.asarray(u)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ShapeError(f"propagator must be a square matrix, got shape {m.shape}")
    d = m.shape[0]
    state = np.asarray(state)
    if state.shape == (d,):
        return apply_batch(m, state[None, :])[0]
    if state.shape == (d, d):
        return apply_batch(m, state[None, :, :])[0]
    raise ShapeError(
        f"state shape {state.shape} matches neither a vector ({d},) "
        f"nor a density matrix ({d}, {d})")


def apply_batch(u, states) -> np.ndarray:
    """``apply`` over a batch: (count, d) state vectors -> U psi_k, or
    (count, d, d) density matrices -> U rho_k U^+, one device call (complex128,
    or complex64 when both U and the states are complex64)."""
    import torch

    m = u.u if isinstance(u, PropagatorResult) else np.asarray(u)
    if m.ndim != 2 or m.shape[0] != m.shape[1]:
        raise ShapeError(f"propagator must be a square matrix, got shape {m.shape}")
    d = m.shape[0]
    states = np.asarray(states)
    if states.ndim == 2 and states.shape[1] == d:
        kind = 0
    elif states.ndim == 3 and states.shape[1:] == (d, d):
        kind = 1
    else:
        raise ShapeError(f"states of shape {states.shape} are neither (count, {d}) vectors nor "
                         f"(count, {d}, {d}) density matrices")
    c64 = m.dtype == np.complex64 and states.dtype == np.complex64
    dtype, tdt, bits = ((np.complex64, torch.complex64, 32) if c64
                        else (np.complex128, torch.complex128, 64))
    count = states.shape[0]
    if count == 0:
        return np.zeros(states.shape, dtype=dtype)
    dev = torch.device("cuda", torch.cuda.current_device())
    du = torch.from_numpy(np.ascontiguousarray(m, dtype=dtype)).to(dev)
    ds = torch.from_numpy(np.ascontiguousarray(states, dtype=dtype)).to(dev)
    out = torch.empty_like(ds)
    nbytes = lib.sp_apply_batch_scratch_bytes(bits, d, count, kind)
    scratch = torch.empty(max(1, nbytes), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    check(lib.sp_apply_batch_device(bits, d, du.data_ptr(), count, kind, ds.data_ptr(),
                                    out.data_ptr(), scratch.data_ptr(), stream.cuda_stream))
    stream.synchronize()
    return out.cpu().numpy()


def reduce_pairwise(batch, backend=None, scratch=None) -> np.ndarray:
    """Time-ordered product U[n-1] ... U[0] of a propagator batch on the
    device (``propagator.py:68-102``): the reference's level-order fold, later
    slices on the left, odd leftovers carried forward; an empty batch gives
    the identity.  ``batch`` is a reference-style batch (anything with a
    ``matrices()`` view) or an (n, d, d) array; the result keeps its complex
    dtype.  ``backend`` and ``scratch`` are accepted for signature
    compatibility (the device owns its scratch)."""
    import torch

    u = batch.matrices() if hasattr(batch, "matrices") else np.asarray(batch)
    if u.ndim != 3 or u.shape[1] != u.shape[2]:
        raise ShapeError(f"expected (n, d, d) matrices, got shape {u.shape}")
    n, d = u.shape[0], u.shape[1]
    out_dtype = np.complex64 if u.dtype == np.complex64 else np.complex128
    if n == 0:
        return np.eye(d, dtype=out_dtype)
    ctx = create("fp32" if out_dtype == np.complex64 else "fp64")
    try:
        ctx.set_hamiltonian(ControlSystem(np.zeros((d, d), dtype=np.complex128)))
        dev = torch.device("cuda", ctx.device)
        mats = torch.from_numpy(np.ascontiguousarray(u, dtype=np.complex128)).to(dev)
        res = torch.empty((d, d), dtype=torch.complex64 if out_dtype == np.complex64
                          else torch.complex128, device=dev)
        stream = torch.cuda.current_stream(dev)
        ctx.product_device_ptr(n, mats.data_ptr(), res.data_ptr(), stream=stream.cuda_stream)
        return res.cpu().numpy()
    finally:
        ctx.close()


class IntegratorContext:
    """Stateful propagation session bound to one B200 (``propagator.py:132-331``).

    Use :func:`create`.  Owns one native context (device scratch, stream);
    independent contexts may coexist.  Not thread-safe, not reentrant.
    """

    def __init__(self, precision: Precision, m_max: int | None, checked: bool, device: int,
                 backend: DeviceBackend | None = None, devices: list[int] | None = None):
        self.precision = precision
        self.m_max = m_max
        self.checked = checked
        # scaling and squaring past the capability (scaling.py); off = the
        # reference's StepTooLargeError
        self.scaling = False
        self.devices = list(devices) if devices else [int(device)]
        self.device = self.devices[0]
        # one batch backend per context (reference: one CpuBackend per
        # context, test_propagator.py:228-238); its name is "b200"
        self.backend = backend if backend is not None else DeviceBackend(device)
        self._state = _CREATED
        self._system: ControlSystem | None = None
        self._effective: EffectiveSystem | None = None
        self._magnus = False
        self._quadrature = Quadrature.MIDPOINT
        handle = ctypes.c_void_p()
        ids = (ctypes.c_int * len(self.devices))(*self.devices)
        check(lib.sp_create(ctypes.byref(handle), precision.bits, len(self.devices), ids))
        self._handle = handle

    # -- lifecycle ---------------------------------------------------------
    @property
    def state(self) -> str:
        return self._state

    @property
    def magnus(self) -> bool:
        return self._magnus

    @property
    def quadrature(self) -> Quadrature:
        return self._quadrature

    @property
    def mode(self) -> str:
        if self._quadrature is Quadrature.GAUSS:  # extension modes
            return "gauss4" if self._magnus else "gauss2"
        if self._magnus:
            return "magnus"
        return self._quadrature.value

    def _require_open(self) -> None:
        if self._state == _CLOSED:
            raise StateMachineError("context is closed")

    def _require_loaded(self) -> None:
        self._require_open()
        if self._state != _LOADED:
            raise StateMachineError("no Hamiltonian loaded; call set_hamiltonian first")

    def set_hamiltonian(self, system: ControlSystem, magnus: bool = False,
                        quadrature=None) -> None:
        """Load (or replace) the system; resolves the slicing mode
        (``propagator.py:175-201``)."""
        self._require_open()
        if not isinstance(system, ControlSystem):
            raise ShapeError(f"expected a ControlSystem, got {type(system).__name__}")
        magnus = bool(magnus)
        if quadrature is None:
            quadrature = Quadrature.SIMPSON if magnus else Quadrature.MIDPOINT
        quadrature = Quadrature.parse(quadrature)
        if magnus and quadrature is Quadrature.MIDPOINT:
            raise ConfigError("the fourth-order mode requires the three-point "
                              "quadrature; midpoint sampling cannot feed it")
        effective = build_effective_system(system) if magnus else None
        terms = effective.terms() if magnus else system.terms()
        stacked = np.ascontiguousarray(np.stack(terms), dtype=np.complex128)
        if quadrature is Quadrature.GAUSS:
            mode = "gauss4" if magnus else "gauss2"  # extension modes
        else:
            mode = "magnus" if magnus else quadrature.value
        check(lib.sp_set_hamiltonian(self._handle, system.dim, system.n_controls,
                                     len(terms), MODE[mode],
                                     stacked.ctypes.data_as(ctypes.c_void_p)), self._handle)
        self._system = system
        self._effective = effective
        self._magnus = magnus
        self._quadrature = quadrature
        self._plan_cache = None  # the bound depends on the system and the mode
        self._state = _LOADED

    def close(self) -> None:
        """Release device storage; further calls raise.  Idempotent."""
        if getattr(self, "_handle", None) is not None and self._handle.value:
            lib.sp_free(self._handle)
            self._handle = ctypes.c_void_p()
        self._system = None
        self._effective = None
        self._state = _CLOSED

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self) -> "IntegratorContext":
        return self

    def __exit__(self, exc_type, exc, tb) -> None:
        self.close()

    # -- host-side preparation (validation order of propagator.py:238-263) --
    def slice_count(self, pts: int) -> int:
        if self._quadrature is Quadrature.GAUSS:
            if pts < 2 or pts % 2:
                raise SamplingParityError(
                    f"Gauss-Legendre quadrature needs an even number of samples >= 2, got {pts}")
            return pts // 2
        if self._quadrature is Quadrature.SIMPSON:
            if pts < 3 or pts % 2 == 0:
                raise SamplingParityError(
                    f"three-point quadrature needs an odd number of samples >= 3, got {pts}")
            return (pts - 1) // 2
        return pts

    def bound(self, dt: float) -> float:
        """Global spectral bound beta for sample step dt (alpha = -beta)."""
        if self._magnus:
            if self._quadrature is Quadrature.GAUSS:
                from .magnus import gauss_magnus_bound
                return gauss_magnus_bound(self._effective, dt)
            return magnus_bound(self._effective, dt)
        step = dt if self._quadrature is Quadrature.MIDPOINT else 2.0 * dt
        return spectral_bound(self._system, step)

    def plan_for(self, dt: float) -> ChebyshevPlan:
        # the plan depends only on dt for a loaded system: the last one is
        # kept (with its native struct) for repeated calls at the same step
        cache = getattr(self, "_plan_cache", None)
        if cache is not None and cache[0] == dt and cache[1] is self._system:
            return cache[2]  # (set_hamiltonian clears the cache)
        beta = self.bound(dt)
        plan = make_plan(-beta, beta, self.precision, m_max=self.m_max)
        self._plan_cache = (dt, self._system, plan, plan.to_native())
        return plan

    def _native_plan(self, plan: ChebyshevPlan):
        cache = getattr(self, "_plan_cache", None)
        if cache is not None and cache[2] is plan:
            return cache[3]
        return plan.to_native()

    def _prepare(self, amps: ControlAmplitudes):
        self._require_loaded()
        if not isinstance(amps, ControlAmplitudes):
            raise ShapeError(f"expected ControlAmplitudes, got {type(amps).__name__}")
        count = self.slice_count(amps.pts)
        if amps.n_controls != self._system.n_controls:
            raise ShapeError(f"amplitude table has {amps.n_controls} controls, "
                             f"system has {self._system.n_controls}")
        # |c| <= 1 is validated inside the lane kernels (no host pass over the
        # table); the host pass runs only where the reference's error
        # precedence needs it before another error can be raised
        try:
            plan = self.plan_for(amps.dt)
        except StepTooLargeError:
            check_pair(self._system, amps)
            raise
        if self.checked:
            check_pair(self._system, amps)
            self._check_hermitian(amps)
        return count, plan

    def _run_checked(self, rc: int, amps: ControlAmplitudes) -> None:
        """Raise the device-side amplitude violation with the reference's
        message (``hamiltonian.py:170-174``), else map the code."""
        if rc == 3:
            idx = ctypes.c_int64(-1)
            lib.sp_amplitude_violation(self._handle, ctypes.byref(idx))
            if idx.value >= 0:
                n = max(1, amps.n_controls)
                k, i = divmod(idx.value, n)
                raise AmplitudeBoundError(
                    f"control amplitude {float(amps.values[k, i])!r} at sample {k}, "
                    f"control {i} lies outside [-1, 1]")
        check(rc, self._handle)

    def _check_hermitian(self, amps: ControlAmplitudes) -> None:
        """checked=True: Hermiticity of every slice exponent in the working
        precision, tolerance 100 u max(1, max|G| d) (``chebyshev.py:249-256``).
        Host-side validation only; the propagation still runs on the GPU."""
        cdt = self.precision.complex_dtype
        terms = [np.asarray(t).astype(cdt) for t in
                 (self._effective.terms() if self._magnus else self._system.terms())]
        v = amps.values
        if self._quadrature is Quadrature.GAUSS:
            from .magnus import gauss_table
            full, scale = gauss_table(amps, self._magnus)
            table = full[:, 1:]
        elif self._magnus:
            from .magnus import magnus_coefficients
            scale = 2.0 * amps.dt
            table = magnus_coefficients(amps) / scale
        elif self._quadrature is Quadrature.SIMPSON:
            c1, c2, c3 = simpson_triplets(v)
            scale = 2.0 * amps.dt
            table = (c1 + 4.0 * c2 + c3) / 6.0
        else:
            scale = amps.dt
            table = v
        d = self._system.dim
        flat = np.stack([t.reshape(d * d) for t in terms])
        asym_t = np.stack([(t - t.conj().T).reshape(d * d) for t in terms])
        asym = gmax = 0.0
        step = max(1, (1 << 20) // max(1, d * d))
        for lo in range(0, table.shape[0], step):
            w = np.column_stack([np.ones(min(step, table.shape[0] - lo)),
                                 table[lo:lo + step]]).astype(cdt)
            g = scale * (w @ flat)
            a = scale * (w @ asym_t)
            gmax = max(gmax, float(np.abs(g).max()))
            asym = max(asym, float(np.abs(a).max()))
        tol = 100.0 * self.precision.roundoff * max(1.0, gmax * d)
        if asym > tol:
            raise HermiticityError(
                f"exponent batch asymmetry {asym:.3g} exceeds tolerance {tol:.3g}")

    # -- propagation --------------------------------------------------------
    def _out_dtype(self):
        return self.precision.complex_dtype

    def equiprop(self, amps: ControlAmplitudes, reduction: str = "pairwise") -> PropagatorResult:
        """Total propagator over the sampled window (``propagator.py:279-308``)."""
        if reduction not in REDUCTION:
            raise ConfigError(f"unknown reduction {reduction!r}; expected pairwise or sequential")
        self._require_loaded()
        if not isinstance(amps, ControlAmplitudes):
            raise ShapeError(f"expected ControlAmplitudes, got {type(amps).__name__}")
        d = self._system.dim
        if amps.pts == 0:
            return PropagatorResult(u=np.eye(d, dtype=self._out_dtype()), slice_count=0,
                                    plan=None)
        try:
            count, plan = self._prepare(amps)
        except StepTooLargeError:
            if not self.scaling:
                raise
            # past the series capability: scaling and squaring (scaling.py)
            from .scaling import equiprop_scaled
            return equiprop_scaled(self, amps, reduction)
        out = np.empty((d, d), dtype=self._out_dtype())
        native = self._native_plan(plan)
        rc = lib.sp_equiprop(self._handle, amps.values.ctypes.data_as(ctypes.c_void_p),
                             amps.pts, amps.n_controls, amps.dt, ctypes.byref(native),
                             REDUCTION[reduction], out.ctypes.data_as(ctypes.c_void_p))
        self._run_checked(rc, amps)
        return PropagatorResult(u=out, slice_count=count, plan=plan.summary())

    def equiprop_all(self, amps: ControlAmplitudes) -> CumulativeResult:
        """Cumulative propagators at every slice boundary (``propagator.py:310-331``)."""
        self._require_loaded()
        if not isinstance(amps, ControlAmplitudes):
            raise ShapeError(f"expected ControlAmplitudes, got {type(amps).__name__}")
        d = self._system.dim
        if amps.pts == 0:
            return CumulativeResult(u_all=np.zeros((0, d, d), dtype=self._out_dtype()),
                                    slice_count=0, plan=None)
        count, plan = self._prepare(amps)
        out = np.empty((count, d, d), dtype=self._out_dtype())
        native = self._native_plan(plan)
        rc = lib.sp_equiprop_all(self._handle, amps.values.ctypes.data_as(ctypes.c_void_p),
                                 amps.pts, amps.n_controls, amps.dt, ctypes.byref(native),
                                 out.ctypes.data_as(ctypes.c_void_p))
        self._run_checked(rc, amps)
        return CumulativeResult(u_all=out, slice_count=count, plan=plan.summary())

    # -- device-resident entry (bench / multi-GPU sharding) -------------------
    def equiprop_device_ptr(self, amps_ptr: int, pts: int, n_ctrl: int, dt: float,
                            out_ptr: int, stream: int = 0, reduction: str = "pairwise",
                            plan: ChebyshevPlan | None = None) -> dict:
        """Asynchronous propagation of a device-resident (pts, n_ctrl) float64
        table into a device d x d output (working dtype).  The caller owns
        amplitude validation (see ``sharding.equiprop_tensor``)."""
        self._require_loaded()
        if reduction not in REDUCTION:
            raise ConfigError(f"unknown reduction {reduction!r}; expected pairwise or sequential")
        if n_ctrl != self._system.n_controls:
            raise ShapeError(f"amplitude table has {n_ctrl} controls, "
                             f"system has {self._system.n_controls}")
        count = self.slice_count(pts) if pts else 0
        plan = plan or self.plan_for(dt)
        native = self._native_plan(plan)
        check(lib.sp_equiprop_device(self._handle, ctypes.c_void_p(amps_ptr), int(pts),
                                     int(n_ctrl), float(dt), ctypes.byref(native),
                                     REDUCTION[reduction], ctypes.c_void_p(out_ptr),
                                     ctypes.c_void_p(stream)), self._handle)
        return {"slice_count": count, "plan": plan.summary()}

    def equiprop_all_device_ptr(self, amps_ptr: int, pts: int, n_ctrl: int, dt: float,
                                out_ptr: int, stream: int = 0,
                                plan: ChebyshevPlan | None = None) -> dict:
        """Asynchronous cumulative propagators of a device-resident (pts,
        n_ctrl) float64 table into a device (slices, d, d) array (working
        dtype).  The caller owns amplitude validation."""
        self._require_loaded()
        if n_ctrl != self._system.n_controls:
            raise ShapeError(f"amplitude table has {n_ctrl} controls, "
                             f"system has {self._system.n_controls}")
        count = self.slice_count(pts) if pts else 0
        plan = plan or self.plan_for(dt)
        native = self._native_plan(plan)
        check(lib.sp_equiprop_all_device(self._handle, ctypes.c_void_p(amps_ptr), int(pts),
                                         int(n_ctrl), float(dt), ctypes.byref(native),
                                         ctypes.c_void_p(out_ptr), ctypes.c_void_p(stream)),
              self._handle)
        return {"slice_count": count, "plan": plan.summary()}

    def product_device_ptr(self, count: int, mats_ptr: int, out_ptr: int, stream: int = 0,
                           reduction: str = "pairwise") -> None:
        """Ordered product mats[count-1] ... mats[0] of device complex128 d x d
        matrices (multi-GPU gather step)."""
        self._require_loaded()
        check(lib.sp_product_device(self._handle, int(count), ctypes.c_void_p(mats_ptr),
                                    REDUCTION[reduction], ctypes.c_void_p(out_ptr),
                                    ctypes.c_void_p(stream)), self._handle)

    def set_scaling(self, enabled: bool = True) -> None:
        """Propagate steps past the series capability by scaling and
        squaring (``scaling.py``) instead of raising ``StepTooLargeError``
        (the reference behaviour, kept by default).  ``equiprop`` only; steps
        within the capability are unaffected."""
        self._require_open()
        self.scaling = bool(enabled)

    _ALGOS = {"auto": 0, "clenshaw": 1, "ps": 2, "ps3m": 3}

    def set_algorithm(self, algo: str = "auto") -> None:
        """Series evaluation scheme: "auto" (Paterson-Stockmeyer in the
        Chebyshev basis when it needs fewer GEMMs per slice), "clenshaw" (the
        reference recurrence, ``chebyshev.py:298-303``) or "ps".  The
        polynomial (plan, truncation) is the same in every case."""
        if algo not in self._ALGOS:
            raise ConfigError(f"unknown algorithm {algo!r}; expected {sorted(self._ALGOS)}")
        check(lib.sp_set_algorithm(self._handle, self._ALGOS[algo]), self._handle)

    def amplitude_violation(self) -> int:
        """Row-major index of the first |c| > 1 (or NaN) sample seen by the
        last device-resident propagation, -1 if none (synchronises)."""
        idx = ctypes.c_int64(-1)
        rc = lib.sp_amplitude_violation(self._handle, ctypes.byref(idx))
        if rc not in (0, 3):
            check(rc, self._handle)
        return idx.value

    def last_algorithm(self) -> dict:
        a = ctypes.c_int()
        g = ctypes.c_int()
        check(lib.sp_last_algorithm(self._handle, ctypes.byref(a), ctypes.byref(g)), self._handle)
        return {"algorithm": {0: "none", 1: "clenshaw", 2: "ps", 3: "ps3m", 4: "clenshaw_fp32"}.get(a.value, "?"),
                "gemms_per_slice": g.value}

    def last_lanes(self) -> int:
        """Lanes of the last lane pass (slices per lane = slices / lanes)."""
        n = ctypes.c_int()
        check(lib.sp_last_lanes(self._handle, ctypes.byref(n)), self._handle)
        return n.value

    def set_profiling(self, enabled: bool = True) -> None:
        check(lib.sp_set_profiling(self._handle, int(bool(enabled))), self._handle)

    def last_timing(self) -> dict:
        ms = ctypes.c_double()
        launches = ctypes.c_int()
        flops = ctypes.c_double()
        name = ctypes.create_string_buffer(128)
        check(lib.sp_last_timing(self._handle, ctypes.byref(ms), ctypes.byref(launches),
                                 ctypes.byref(flops), name, 128), self._handle)
        return {"main_kernel_ms": ms.value, "launches": launches.value,
                "executed_flops": flops.value, "kernel": name.value.decode()}


def _default_device() -> int:
    for key in ("SLICEPROP_DEVICE", "LOCAL_RANK"):
        if os.environ.get(key, "").isdigit():
            return int(os.environ[key])
    return 0


def create(precision="fp64", m_max: int | None = None, checked: bool = False,
           backend=None, device: int | None = None,
           devices=None, scaling: bool = False) -> IntegratorContext:
    """New propagation context (``propagator.py:334-355``) on one B200, or
    on several in this one process: ``devices=[0, 1, ...]`` (or an int
    count) time-shards every ``equiprop`` over those GPUs — contiguous slice
    blocks, one per device, block products gathered on ``devices[0]`` by
    peer copies and multiplied in time order.

    precision "fp32" | "fp64"; m_max pins the series order (odd 3..25);
    checked enables the Hermiticity sanity pass.  backend accepts None, a
    ``DeviceBackend`` instance or a GPU token ("b200", "cuda", "gpu",
    "sm_100a") — the reference's "cpu" backend is not offered: this package
    has no CPU path.
    """
    precision = Precision.parse(precision)
    if m_max is not None and m_max not in ORDER_GRID:
        raise ConfigError(f"m_max override {m_max} not an odd integer in "
                          f"{ORDER_GRID[0]}..{ORDER_GRID[-1]}")
    dev = _default_device() if device is None else int(device)
    if devices is not None:
        devices = list(range(int(devices))) if isinstance(devices, int) else \
            [int(x) for x in devices]
        if not devices or any(x < 0 for x in devices) or len(devices) > 64:
            raise ConfigError(f"devices must be 1..64 non-negative ordinals, got {devices!r}")
        dev = devices[0]
    instance = None
    if isinstance(backend, DeviceBackend):
        instance, dev = backend, backend.device if device is None else dev
    elif backend is not None:
        if not isinstance(backend, str) or backend.lower() not in _BACKEND_TOKENS:
            raise ConfigError(f"unknown backend {backend!r}; expected one of {_BACKEND_TOKENS}")
    ctx = IntegratorContext(precision, m_max, bool(checked), dev, instance, devices)
    ctx.scaling = bool(scaling)
    return ctx
