"""ORACLE — test infrastructure, not product code.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything under ``oracle/``.  It shares no
code with ``paper_1507_06078_b200`` (the CUDA path) and never imports it; the
only shared module is ``synth`` (seeded inputs, no method arithmetic).

A plain, slow, fp64 CPU implementation of what the hot path computes, written
from arXiv 1507.06078 (PAPER.md = P):

* sparse part in plain C (``csr_oracle.c``: SpMM, Chebyshev filter, column
  norms), loaded with ctypes;
* dense part in ``dense.py``: the oracle's own pivoted / blocked Householder QR,
  cyclic Jacobi eig, Cholesky and Gaussian elimination (no LAPACK on the oracle
  path; numpy matmul serves as a single library step of the tall-skinny products).

Every function cites the passage it follows.  The pins that tie it to the
paper and to mathematics (not to itself) are in ``tests/test_oracle_*.py``.
Functions without such a pin are marked "parity unpinned" — currently none.
"""
from .core import (  # noqa: F401
    load_lib,
    spmm,
    cheb_filter,
    col_norms,
    mpm_sweep,
    gershgorin_lower,
    chebyshev_T,
    interp_coeffs,
    psi,
    poly_filter,
    poly_sweep,
    gn_step,
    orthonormalize,
    rayleigh_ritz,
    arr,
    residuals,
    sweeps_rule,
    RANGE_DIGITS,
    solve,
    solve_deflate,
    rcond_gram,
    SolveResult,
)
from . import dense  # noqa: F401
