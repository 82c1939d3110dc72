"""GP-FVM oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the CUDA path
computes, written from PAPER.md (arxiv 2406.05020).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product path
(``paper_2406_05020_b200``) never imports it and shares no code with it; both
consume the seeded problem descriptions of ``gpfvm_inputs`` only.

Modules
  matern.py     1D half-integer Matérn calculus (§3.1, Eq. 12, l.213-220)
                in mpmath at 40 significant digits, rounded to fp64 at the end.
  gram.py       1D functionals (Eq. 10, l.207), factor matrices (Eq. 16/20,
                l.244-246, l.318), dense Gram assembly and the plain Kronecker
                matvec (Eq. 20, l.316-320) in fp64.
  solve.py      dense Cholesky solve (§4, l.289), IterGP/CG with full
                reorthogonalisation (§4.1, l.295-302; §6 l.475) and the
                preconditioner defined in DESIGN.md §5.
  posterior.py  posterior mean / variance (Eqs. 5-6, l.113-114) on tensor grids.

Pins (tests that tie the oracle to something other than itself) live in
``tests/test_oracle_*.py``.  Parity status per function is listed in
DESIGN.md §3; every function here is pinned (no "parity unpinned" entries).
"""
