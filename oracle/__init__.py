"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the equiprop hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed CPU baseline.  The product package
``paper_2108_07126_b200`` never imports it: its propagation path is the
sm_100a CUDA library and fails loudly when that library is missing.

Parity is pinned: ``tests/golden/make_golden.py`` generated the committed
fixtures by importing the reference (``/root/reference/pkg/src/sliceprop``)
in the build container, and ``tests/test_oracle.py`` checks this restatement
against every fixture (bit-for-bit for the host plan and for the
propagators, since both run the same numpy operation sequence).
"""

from .sliceprop_oracle import *  # noqa: F401,F403
from .sliceprop_oracle import __all__  # noqa: F401
