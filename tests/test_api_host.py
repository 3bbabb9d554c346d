"""Host-side contract of the drop-in API (no GPU needed): lifecycle, mode
resolution, validation order and error codes, mirroring the reference tests
(tests/test_propagator.py TestLifecycle/TestEquiprop error cases,
tests/test_hamiltonian.py, bindings/tests/test_binding.py error mapping).

Every check here fails BEFORE the device is touched; the one call that
reaches the device asserts the loud no-GPU failure (no CPU fallback).
"""

import numpy as np
import pytest

import paper_2108_07126_b200 as sp
from paper_2108_07126_b200 import pysliceprop

SZ = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=complex)
SX = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)
SY = np.array([[0.0, -1.0j], [1.0j, 0.0]], dtype=complex)


def drift_qubit():
    return sp.ControlSystem(SZ / 2.0)


def driven_qubit():
    return sp.ControlSystem(SZ / 2.0, [SX / 2.0, SY / 2.0])


def driven_amps(pts, dt=0.02):
    t = np.arange(pts) * dt
    return sp.ControlAmplitudes(np.column_stack([np.cos(t), np.sin(t)]), dt)


def _gpu_present():
    import ctypes
    n = ctypes.c_int(0)
    sp._native.lib.sp_device_count(ctypes.byref(n))
    return n.value > 0


class TestLifecycle:
    def test_create_defaults(self):
        ctx = sp.create()
        assert ctx.state == "created"
        assert ctx.precision.value == "fp64"
        assert ctx.backend.name == "b200"

    def test_invalid_tokens(self):
        with pytest.raises(sp.ConfigError):
            sp.create(precision="fp16")
        with pytest.raises(sp.ConfigError):
            sp.create(m_max=4)
        with pytest.raises(sp.ConfigError):
            sp.create(m_max=27)
        with pytest.raises(sp.ConfigError):
            sp.create(backend="cpu")
        assert sp.create(backend="b200").backend.name == "b200"

    def test_propagate_before_load(self):
        ctx = sp.create()
        amps = sp.ControlAmplitudes(np.zeros((4, 0)), 0.1)
        with pytest.raises(sp.StateMachineError):
            ctx.equiprop(amps)
        with pytest.raises(sp.StateMachineError):
            ctx.equiprop_all(amps)

    def test_closed_context_rejects_everything(self):
        ctx = sp.create()
        ctx.set_hamiltonian(drift_qubit())
        ctx.close()
        amps = sp.ControlAmplitudes(np.zeros((4, 0)), 0.1)
        with pytest.raises(sp.StateMachineError):
            ctx.equiprop(amps)
        with pytest.raises(sp.StateMachineError):
            ctx.equiprop_all(amps)
        with pytest.raises(sp.StateMachineError):
            ctx.set_hamiltonian(drift_qubit())
        ctx.close()
        assert ctx.state == "closed"

    def test_context_manager_closes(self):
        with sp.create() as ctx:
            ctx.set_hamiltonian(drift_qubit())
            assert ctx.state == "loaded"
        assert ctx.state == "closed"

    def test_magnus_mode_resolution(self):
        ctx = sp.create()
        with pytest.raises(sp.ConfigError):
            ctx.set_hamiltonian(driven_qubit(), magnus=True, quadrature="midpoint")
        ctx.set_hamiltonian(driven_qubit(), magnus=True)
        assert ctx.quadrature.value == "simpson"
        assert ctx.mode == "magnus"
        with pytest.raises(sp.ConfigError):
            ctx.set_hamiltonian(driven_qubit(), quadrature="trapezoid")

    def test_rejects_non_system(self):
        with pytest.raises(sp.ShapeError):
            sp.create().set_hamiltonian(np.eye(2))


class TestValidation:
    def test_empty_table_is_identity_without_device(self):
        ctx = sp.create()
        ctx.set_hamiltonian(driven_qubit())
        res = ctx.equiprop(sp.ControlAmplitudes(np.zeros((0, 2)), 0.1))
        assert np.array_equal(res.u, np.eye(2)) and res.slice_count == 0 and res.plan is None
        cum = ctx.equiprop_all(sp.ControlAmplitudes(np.zeros((0, 2)), 0.1))
        assert cum.u_all.shape == (0, 2, 2) and np.array_equal(cum.final, np.eye(2))
        ctx32 = sp.create(precision="fp32")
        ctx32.set_hamiltonian(driven_qubit())
        assert ctx32.equiprop(sp.ControlAmplitudes(np.zeros((0, 2)), 0.1)).u.dtype == np.complex64

    def test_unknown_reduction(self):
        ctx = sp.create()
        ctx.set_hamiltonian(drift_qubit())
        with pytest.raises(sp.ConfigError):
            ctx.equiprop(sp.ControlAmplitudes(np.zeros((2, 0)), 0.1), reduction="tree")

    def test_rejects_raw_arrays(self):
        ctx = sp.create()
        ctx.set_hamiltonian(drift_qubit())
        with pytest.raises(sp.ShapeError):
            ctx.equiprop(np.zeros((4, 0)))

    def test_control_count_mismatch(self):
        ctx = sp.create()
        ctx.set_hamiltonian(driven_qubit())
        with pytest.raises(sp.ShapeError):
            ctx.equiprop(sp.ControlAmplitudes(np.zeros((4, 1)), 0.1))

    def test_amplitude_validation_host_utility(self):
        # equiprop validates |c| <= 1 inside the lane kernels (GPU test:
        # tests/test_api_gpu.py); the reference's host utility is kept
        values = np.zeros((4, 2))
        values[2, 1] = 1.5
        values[3, 0] = 7.0
        v = sp.validate_amplitudes(sp.ControlAmplitudes(values, 0.1))
        assert (v.sample, v.control, v.value) == (2, 1, 1.5)
        values[2, 1] = np.nan
        assert sp.validate_amplitudes(sp.ControlAmplitudes(values, 0.1)).sample == 2

    def test_step_too_large_keeps_amplitude_precedence(self):
        # reference order: amplitude check before the plan (hamiltonian.py:197)
        ctx = sp.create()
        ctx.set_hamiltonian(driven_qubit())
        values = np.zeros((4, 2))
        values[1, 0] = 3.0
        with pytest.raises(sp.AmplitudeBoundError, match="sample 1, control 0"):
            ctx.equiprop(sp.ControlAmplitudes(values, 100.0))

    def test_parity_enforced_before_amplitudes(self):
        ctx = sp.create()
        ctx.set_hamiltonian(driven_qubit(), quadrature="simpson")
        bad = np.full((4, 2), 2.0)
        with pytest.raises(sp.SamplingParityError):
            ctx.equiprop(sp.ControlAmplitudes(bad, 0.1))
        with pytest.raises(sp.SamplingParityError):
            ctx.equiprop(driven_amps(1))
        ctx.set_hamiltonian(driven_qubit(), magnus=True)
        with pytest.raises(sp.SamplingParityError):
            ctx.equiprop(driven_amps(10))

    def test_step_too_large_carries_remedy(self):
        ctx = sp.create()
        ctx.set_hamiltonian(drift_qubit())
        with pytest.raises(sp.StepTooLargeError) as ei:
            ctx.equiprop(sp.ControlAmplitudes(np.zeros((3, 0)), 10.0))
        assert ei.value.norm_bound == pytest.approx(5.0)
        assert ei.value.capability == pytest.approx(sp.norm_capability(25, "fp64"))

    def test_plan_records_selected_order(self):
        ctx = sp.create()
        ctx.set_hamiltonian(drift_qubit())
        plan = ctx.plan_for(0.1)
        assert plan.beta == pytest.approx(0.05) and plan.alpha == pytest.approx(-0.05)
        assert plan.m_max == 7 and 0.0 < plan.predicted_error < 2.0 ** -53
        assert sp.create(m_max=13).__class__ is sp.IntegratorContext

    def test_checked_mode_rejects_non_hermitian_exponent(self):
        h = np.array([[0.0, 1.0], [1.0 + 5e-13, 0.0]], dtype=complex)  # passes ingest
        ctx = sp.create(checked=True)
        ctx.set_hamiltonian(sp.ControlSystem(h, [h]))
        with pytest.raises(sp.HermiticityError):
            ctx.equiprop(sp.ControlAmplitudes(np.ones((3, 1)), 0.1))

    @pytest.mark.skipif(_gpu_present(), reason="asserts the no-GPU failure mode")
    def test_no_gpu_fails_loudly(self):
        ctx = sp.create()
        ctx.set_hamiltonian(driven_qubit())
        with pytest.raises(sp.InternalError, match="no CPU fallback"):
            ctx.equiprop(driven_amps(5))


class TestSystemModel:
    def test_ingest(self, rng):
        h = rng.standard_normal((3, 3)) + 1j * rng.standard_normal((3, 3))
        with pytest.raises(sp.HermiticityError):
            sp.ControlSystem(h)
        with pytest.raises(sp.ShapeError):
            sp.ControlSystem(np.zeros((2, 3)))
        with pytest.raises(sp.ShapeError):
            sp.ControlSystem(np.eye(2), [np.eye(3)])
        sys_ = sp.ControlSystem(SZ, [SX])
        assert sys_.norms == (1.0, 1.0) and sys_.n_controls == 1

    def test_amplitudes(self):
        with pytest.raises(sp.ConfigError):
            sp.ControlAmplitudes(np.zeros((3, 1)), 0.0)
        with pytest.raises(sp.ShapeError):
            sp.ControlAmplitudes(np.zeros(3), 0.1)
        a = sp.ControlAmplitudes(np.zeros((3, 2)), 0.1)
        assert not a.values.flags.writeable and a.n_controls == 2

    def test_effective_system_ordering(self):
        eff = sp.build_effective_system(driven_qubit())
        assert eff.n_effective == 5
        assert np.allclose(eff.effective_controls[2], 1j * sp.commutator(SZ / 2, SX / 2))
        for h in eff.effective_controls:
            assert np.allclose(h, h.conj().T)

    def test_manifest_roundtrip(self, tmp_path):
        import json
        doc = {"dim": 2, "dt": 0.1, "drift": sp.matrix_to_pairs(SZ),
               "controls": [sp.matrix_to_pairs(SX)],
               "amplitudes": {"pts": 3, "data": [[0.1], [0.2], [0.3]]}}
        p = tmp_path / "m.json"
        p.write_text(json.dumps(doc))
        system, amps, prec = sp.load_manifest(str(p))
        assert system.dim == 2 and amps.pts == 3 and prec.value == "fp64"


class TestBindingErrors:
    def test_unknown_mode_keyword(self):
        with pytest.raises(pysliceprop.BindingError) as ei:
            pysliceprop.equiprop(SZ, [], np.zeros((2, 0)), 0.1, bogus=True)
        assert ei.value.code == "config"

    def test_error_codes_preserved(self):
        with pysliceprop.Session() as s:
            with pytest.raises(pysliceprop.BindingError) as ei:
                s.equiprop(np.zeros((3, 0)), 0.1)
            assert ei.value.code == "state-machine"
            s.set_hamiltonian(SZ / 2, [SX / 2], magnus=True)
            with pytest.raises(pysliceprop.BindingError) as ei:
                s.equiprop(np.zeros((4, 1)), 0.1)
            assert ei.value.code == "sampling-parity"
            with pytest.raises(pysliceprop.BindingError) as ei:
                s.equiprop(np.zeros((5, 2)), 0.1)
            assert ei.value.code == "shape"
            with pytest.raises(pysliceprop.BindingError) as ei:
                s.set_hamiltonian(np.array([[0, 1], [2, 0]]), [])
            assert ei.value.code == "hermiticity"
        with pytest.raises(pysliceprop.BindingError) as ei:
            s.equiprop(np.zeros((3, 0)), 0.1)
        assert ei.value.code == "state-machine"
        with pytest.raises(pysliceprop.BindingError) as ei:
            pysliceprop.Session(precision="fp8")
        assert ei.value.code == "config"

    def test_reentrancy_guard(self, monkeypatch):
        s = pysliceprop.Session()
        s.set_hamiltonian(SZ / 2, [])
        seen = {}

        def hijack(*a, **k):
            try:
                s.set_hamiltonian(SZ, [])
            except pysliceprop.BindingError as exc:
                seen["code"] = exc.code
            raise sp.ShapeError("stop")

        monkeypatch.setattr(s._ctx, "equiprop", hijack)
        with pytest.raises(pysliceprop.BindingError):
            s.equiprop(np.zeros((2, 0)), 0.1)
        assert seen["code"] == "state-machine"
        s.close()
        assert s.closed


def test_plan_cache_follows_the_loaded_system():
    """The host caches the last plan per step size; set_hamiltonian clears
    it (the bound depends on the system and the mode)."""
    sz = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=complex)
    sx = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)
    ctx = sp.create()
    ctx.set_hamiltonian(sp.ControlSystem(sz / 2, [sx / 2]))
    p1 = ctx.plan_for(0.1)
    assert ctx.plan_for(0.1) is p1
    assert ctx.plan_for(0.2).beta == pytest.approx(2 * p1.beta)
    ctx.set_hamiltonian(sp.ControlSystem(sz / 2, [sx / 2]), magnus=True)
    p2 = ctx.plan_for(0.1)
    assert p2 is not p1 and p2.beta != p1.beta
    ctx.set_hamiltonian(sp.ControlSystem(2 * sz, [sx / 2]))
    assert ctx.plan_for(0.1).beta > p1.beta
    ctx.close()
