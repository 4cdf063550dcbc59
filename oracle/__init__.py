"""Independent CPU oracle for the LeanVec-Sphering / GleanVec search hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything
under `oracle/`.  The product path (package `paper_2410_22347_b200`) never
imports it, and this package never imports the product; the two share no
code, only the seeded inputs of `lvgen`.

Plain numpy, fp64, written in the paper's order and notation; every function
cites the PAPER.md passage it follows (P:n = PAPER.md line n, S:n = SPEC.md
line n).  Pins live in tests/test_oracle_pins.py.  Parity status per function
is listed in DESIGN.md §4 ("parity unpinned" marks the ones without a pin).
"""
from .lv_oracle import *  # noqa: F401,F403
