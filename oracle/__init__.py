"""CPU oracle for the IRK stage-solve path -- TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy, the algorithm of the reference
package ``irkit`` (``/root/reference/pkg/src/irkit``) for the hot path named
by BASELINE.json: the Newton-like outer loop over the s-stage Gauss/Radau
system, the real-Schur stage decoupling, and block-2x2 preconditioned GMRES
with damped-Jacobi ``(gamma*M - dt*L)`` inner solves.  Every function cites
the reference ``file:line`` it follows.

It is the *checker*, never the thing measured or shipped: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
``paper_2101_01776_b200`` never imports anything from here and fails loudly
when its CUDA extension is missing.

Parity pinning: the restatement is checked against outputs of the real
reference run in the build container (``tests/golden/make_golden.py`` writes
the fixtures under ``tests/golden/``) and against the reference's own
known-answer tests (restated in ``tests/test_oracle.py``).
"""
