"""CPU oracle for TP-Aware Dequantization (arxiv 2402.04925).  TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2402_04925_b200``) never imports it, and this package never imports the
product path: the two share no code (only ``synth`` -- seeded random draws, no
method arithmetic -- feeds both).

Everything is plain numpy in float64, written in the paper's order and notation:
see ``oracle/tp_dequant.py``.  Each function cites the passage it follows.
Pins (tests/test_oracle_pins.py, ``-m "not gpu"``) tie every function to the paper's
worked examples, closed forms, brute force on tiny inputs and exact-arithmetic
identities; no function is "parity unpinned".
"""
from .tp_dequant import *  # noqa: F401,F403
