"""The shared library has no unresolved C++ symbols of its own (a template
declared/defined with mismatching signatures would otherwise only fail when
the library is loaded)."""

import re
import subprocess

from paper_2108_07126_b200 import _native


def test_no_undefined_internal_symbols():
    out = subprocess.run(["nm", "-D", "--undefined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    bad = [ln for ln in out.splitlines() if re.search(r"(engine_cu|sp_ctx|N2sp)", ln)]
    assert not bad, bad
