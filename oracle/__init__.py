"""CPU oracle for the partial-fraction exp(A)V hot path — TEST INFRASTRUCTURE ONLY.

Nothing in the product (`paper_2306_16778_b200`) imports this package.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline / reference arm
may use it, and only as the checker or the timed CPU baseline.

Contents
  restate.py   numpy/scipy restatement of the reference engine
               (/root/reference/pkg/src/pfexpm/engine.py:178-230) for dense
               inputs, plus the structured restatements for C2 (tridiagonal,
               LAPACK zgtsv) and C5 (banded, LAPACK zgbsv) that the dense-only
               reference cannot express.
  closed.py    exact oracles: eigen-decomposition U e^L U^H (linalg.py:120-123)
               and the DST-I closed form for the Dirichlet Laplacians.

Pinning: the reference ships no golden vectors, so
tests/golden/make_golden.py runs the reference itself here and freezes its
tables and outputs; tests/test_oracle.py checks this restatement against them
(pole tables bit-exact, dense outputs bitwise or to 1e-15).  The structured
restatements share the table, pairing and ascending reduction with the dense
one and are pinned through the dense path on small Laplacians (the same matrix
solved densely by the reference and by zgtsv/zgbsv here).
"""
