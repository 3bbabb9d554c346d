"""CLI front end (reference tests/test_cli.py equivalents).  bounds and the
error exit codes run on CPU; propagate/converge need the B200."""

import json
import subprocess
import sys

import numpy as np
import pytest

import paper_2108_07126_b200 as sp
from paper_2108_07126_b200 import cli

SZ = np.array([[1.0, 0.0], [0.0, -1.0]], dtype=complex)
SX = np.array([[0.0, 1.0], [1.0, 0.0]], dtype=complex)


def manifest(tmp_path, dt=0.1, data=None):
    doc = {"dim": 2, "dt": dt, "precision": "fp64", "drift": sp.matrix_to_pairs(SZ / 2),
           "controls": [sp.matrix_to_pairs(SX / 2)],
           "amplitudes": {"pts": 5, "data": data or [[0.1], [0.2], [0.3], [0.2], [0.1]]}}
    p = tmp_path / "m.json"
    p.write_text(json.dumps(doc))
    return str(p)


def test_bounds_table(capsys):
    assert cli.main(["bounds"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "precision,m,bound"
    assert "fp64,25,4.447" in out and "fp32,3,0.033" in out and "fp64,3,2e-04" in out


def test_step_too_large_exit_code(tmp_path, capsys):
    assert cli.main(["propagate", manifest(tmp_path, dt=100.0)]) == 3
    assert "step-too-large" in capsys.readouterr().err


def test_bad_manifest_exit_code(tmp_path, capsys):
    p = tmp_path / "bad.json"
    p.write_text("{}")
    assert cli.main(["propagate", str(p)]) == 2


def test_module_entry_point():
    proc = subprocess.run([sys.executable, "-m", "paper_2108_07126_b200", "bounds",
                           "--precision", "fp32"], capture_output=True, text=True)
    assert proc.returncode == 0 and "fp32,25,9.919" in proc.stdout


@pytest.mark.gpu
def test_propagate_matches_library(tmp_path, capsys):
    path = manifest(tmp_path)
    assert cli.main(["propagate", path, "--all"]) == 0
    doc = json.loads(capsys.readouterr().out)
    u = sp.matrix_from_pairs(doc["u"], "u")
    system, amps, _ = sp.load_manifest(path)
    ctx = sp.create()
    ctx.set_hamiltonian(system)
    assert np.abs(u - ctx.equiprop_all(amps).final).max() <= 1e-15
    assert doc["slice_count"] == 5 and len(doc["u_all"]) == 5


@pytest.mark.gpu
def test_converge_subcommand(capsys):
    assert cli.main(["converge", "--steps-list", "10,32,100,316,1000", "--skip-oracle"]) == 0
    cap = capsys.readouterr()
    assert cap.out.splitlines()[0] == "pts,error"
    assert "fitted order" in cap.err
