"""CPU oracle for the sketched flexible Golub-Kahan step (sFLSQR / sFLSMR).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import, call,
link or execute anything under ``oracle/``.  The product path
(``paper_2605_22281_b200``) never imports it and shares no code with it.

Plain, slow, fp64: NumPy for vector algebra, a plain single-threaded C CSR
product (``csrc/oracle_csr.c``, -ffp-contract=off), Householder QR written out
(``lsq.py``), Philox4x32-10 written out from its published definition
(``philox.py``).  Every function cites the PAPER.md passage it follows; the
readings of paper-silent points are listed in DESIGN.md.

Parity pins (tests/test_oracle_*.py, ``-m "not gpu"``): Philox known-answer
vectors; sketch table properties; Householder vs numpy.linalg.lstsq;
reductions to SciPy LSQR/LSMR (tau = id, S = I, full window); fixed-diagonal
tau vs LSQR on A D^{1/2}; AB-/BA-GMRES brute force for unmatched B; the
Remark sFLSMR == sFLSQR with sketch S A^T; rank-k exactness; Theorem 2.1's
identity; FGK relations; the IRN weights against the IRLS definitions they
implement (the weighted 2-norm tends to the l_p norm, the weights are the
gradient of the smoothed l_p penalty, p = 2 gives no reweighting) and the
NONNEG weights against the properties of a multiplicative nonnegativity
scaling (tests/test_oracle_precond.py; readings R7/R8).
"""
