"""INTEGRATION.md's binding, executed inside a copy of the reference package.

The UNMODIFIED reference (baseline/_ref/sliceprop, tools/install_reference.sh)
is copied to a temp dir and ``integration/sliceprop_b200.py`` is added to it
as ``sliceprop/b200.py`` — exactly what a maintainer would do.  Then:

* the reference's own propagator tests (TestEquiprop, TestMagnusMode,
  TestEquipropAll, TestLifecycle of ``tests/test_propagator.py``) run with
  ``create()`` routed to the B200 backend (``b200.install(default=True)``),
  minus the CPU-backend cost-contract tests;
* ``create(backend="b200")`` results are compared with the same package's
  CPU path on the same inputs, for every mode and both precisions, and with
  a two-device (emulated) native context.
"""

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
LIB = os.path.join(ROOT, "paper_2108_07126_b200", "libsliceprop_b200.so")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(
    not os.path.isdir(os.path.join(REF, "ref_tests", "core")),
    reason="reference not staged (run tools/install_reference.sh)")]

DESELECT = [
    "test_propagator.py::TestEquiprop::test_gemm_budget",
    "test_propagator.py::TestEquiprop::test_scratch_reused_between_calls",
    "test_propagator.py::TestLifecycle::test_backend_tokens",
]

COMPARE = r'''
import numpy as np
import sliceprop
from sliceprop import b200
b200.install()
rng = np.random.default_rng(5)

def herm(d):
    a = rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))
    h = (a + a.conj().T) / 2
    return h / np.abs(h).sum(axis=0).max()

worst = 0.0
for d, n, pts, mode, prec in [(2, 2, 1001, "midpoint", "fp64"), (4, 3, 401, "simpson", "fp64"),
                              (8, 2, 301, "magnus", "fp64"), (32, 2, 200, "midpoint", "fp64"),
                              (128, 4, 41, "midpoint", "fp64"), (2, 2, 1001, "magnus", "fp32"),
                              (16, 2, 201, "simpson", "fp32")]:
    system = sliceprop.ControlSystem(herm(d), [herm(d) for _ in range(n)])
    amps = sliceprop.ControlAmplitudes(rng.uniform(-1, 1, (pts, n)), 0.5 / (n + 1))
    res = {}
    for backend in (None, "b200"):
        with sliceprop.create(precision=prec, backend=backend) as ctx:
            ctx.set_hamiltonian(system, magnus=mode == "magnus",
                                quadrature=None if mode == "magnus" else mode)
            res[backend] = (ctx.equiprop(amps), ctx.equiprop(amps, reduction="sequential"),
                            ctx.equiprop_all(amps))
    cpu, gpu = res[None], res["b200"]
    assert type(gpu[0]) is type(cpu[0]) and gpu[0].plan == cpu[0].plan
    assert gpu[0].slice_count == cpu[0].slice_count and gpu[0].u.dtype == cpu[0].u.dtype
    eps = np.linalg.norm(cpu[0].u - cpu[1].u) / np.linalg.norm(cpu[0].u)
    tol = max(1e-12 if prec == "fp64" else 1e-5, 4 * eps)
    for k in (0, 1):
        err = np.linalg.norm(gpu[k].u - cpu[k].u) / np.linalg.norm(cpu[k].u)
        worst = max(worst, err / tol)
        assert err <= tol, (d, mode, prec, k, err, tol)
    assert gpu[2].u_all.shape == cpu[2].u_all.shape
    assert np.array_equal(gpu[2].u_all[-1], gpu[1].u)
# the backend on two (emulated) devices of this process
sys_ = sliceprop.ControlSystem(herm(64), [herm(64), herm(64)])
amps = sliceprop.ControlAmplitudes(rng.uniform(-1, 1, (500, 2)), 0.1)
ctx = sliceprop.create()
ctx.set_hamiltonian(sys_)
ref = ctx.equiprop(amps).u
ctx.backend = b200.B200Backend(ctx.precision, devices=(0, 0))
ctx.set_hamiltonian(sys_)
got = ctx.equiprop(amps).u
assert np.linalg.norm(got - ref) / np.linalg.norm(ref) <= 1e-12
print("INTEGRATION-OK worst err/tol %.3f" % worst)
'''

CONFTEST = '''
import sliceprop.b200
sliceprop.b200.install(default=True)
'''


def _stage(tmp_path):
    pkg = tmp_path / "pkg"
    shutil.copytree(os.path.join(REF, "sliceprop"), pkg / "sliceprop")
    shutil.copy(os.path.join(ROOT, "integration", "sliceprop_b200.py"),
                pkg / "sliceprop" / "b200.py")
    env = dict(os.environ, SLICEPROP_B200_LIB=LIB)
    env["PYTHONPATH"] = os.pathsep.join([str(pkg), os.path.join(REF, "ref_tests", "core")])
    env.pop("PYTEST_ADDOPTS", None)
    return pkg, env


def test_backend_matches_the_reference_cpu_path(tmp_path):
    _, env = _stage(tmp_path)
    r = subprocess.run([sys.executable, "-c", COMPARE], env=env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0 and "INTEGRATION-OK" in r.stdout, r.stdout + r.stderr[-4000:]
    print(r.stdout.strip())


def test_reference_propagator_tests_on_the_b200_backend(tmp_path):
    _, env = _stage(tmp_path)
    run = tmp_path / "run"
    run.mkdir()
    for f in ("test_propagator.py", "helpers.py", "conftest.py"):
        shutil.copy(os.path.join(REF, "ref_tests", "core", f), run / f)
    (run / "conftest.py").write_text((run / "conftest.py").read_text() + CONFTEST)
    args = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-o", "addopts=",
            "--rootdir", str(run), "test_propagator.py", "-k",
            "TestEquiprop or TestMagnusMode or TestEquipropAll or TestLifecycle"]
    for d in DESELECT:
        args += ["--deselect", d]
    r = subprocess.run(args, cwd=str(run), env=env, capture_output=True, text=True, timeout=900)
    print(r.stdout[-800:])
    assert r.returncode == 0, r.stdout[-5000:] + r.stderr[-2000:]
