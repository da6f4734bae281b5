"""CPU ORACLE — test infrastructure only.

Plain, slow, obviously-correct NumPy (float64 / complex128) implementation of
what the Z_bc coupling hot path of arXiv 2206.12409 computes.  Each function
cites the PAPER.md passage (``P:L``) or the SURVEY.md reading (``§8c-Lx``) it
follows.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from here.
The product path (``paper_2206_12409_b200``) never imports it and shares no
code with it; the only shared module is ``synth`` (seeded inputs, no method
arithmetic).

Parity status per function: every exported function is pinned by a
``-m "not gpu"`` test in ``tests/test_oracle_pins.py`` against a closed form,
an extended-precision value, a textbook special case, an invariant, or brute
force.  No function is "parity unpinned".
"""
from . import geometry, greens, entries, ttmv, ttsvd, maxvol, ttcross, validate  # noqa: F401
