"""Oracle pins for the full fixed-parameter ARRABIT-MPM iteration (SURVEY.md
§8c-3): converged eigenvalues against closed-form spectra, Weyl bounds and a
dense numpy eigensolve; every residual <= tol (Eq. out-stop)."""
import numpy as np
import pytest

import oracle
import synth
from synth import configs


def _check(res, ref, k, tol=1e-10):
    assert res.converged
    assert np.all(res.res <= tol)
    rel = np.abs(res.mu - ref[:k]) / np.maximum(1, np.abs(ref[:k]))
    assert rel.max() < 1e-10, rel.max()
    # partial-trace monitor
    assert abs(res.mu.sum() - ref[:k].sum()) < 1e-9 * abs(ref[:k].sum())


def test_solve_cfg1_closed_form():
    A, spec = configs.build_config(1)
    X0 = synth.starting_block(spec)
    r = oracle.solve(A, spec.k, spec.d, spec.p, X0, tol=spec.tol)
    n = A.n
    lam = np.sort(2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))[::-1]
    _check(r, lam, spec.k)
    # survey's closed-form partial trace
    assert r.mu.sum() == pytest.approx(79.99292600087112, rel=1e-13)


def test_solve_small_lap2d_closed_form():
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    N = spec.size
    c = 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    lam = np.sort((4 - c[:, None] - c[None, :]).ravel())[::-1]
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec))
    _check(r, lam, spec.k)


def test_solve_small_st27_closed_form():
    spec = configs.SMALL_ANALOGS["st27"]
    A, _ = configs.build_config(spec)
    N = spec.size
    t = 1 + 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    lam = np.sort((27 - t[:, None, None] * t[None, :, None] * t[None, None, :]).ravel())[::-1]
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec))
    _check(r, lam, spec.k)


def test_solve_small_lap3d_potential_weyl_and_dense():
    spec = configs.SMALL_ANALOGS["lap3dV"]
    A, _ = configs.build_config(spec)
    N = spec.size
    c = 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    L = np.sort((6 - c[:, None, None] - c[None, :, None] - c[None, None, :]).ravel())[::-1]
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec))
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1]
    _check(r, lam, spec.k)
    # Weyl: lambda_i(L) <= lambda_i(L+V) <= lambda_i(L) + max V
    assert np.all(r.mu >= L[:spec.k] - 1e-12) and np.all(r.mu <= L[:spec.k] + 1 + 1e-12)


def test_solve_small_zipf_dense():
    spec = configs.SMALL_ANALOGS["zipf"]
    A, _ = configs.build_config(spec)
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec))
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1]
    _check(r, lam, spec.k)


def test_solve_smallest_via_negated_matrix_1d_closed_form():
    """The paper's second mode (k smallest, Table 6) = the k largest of -A;
    1-D Laplacian closed form lambda_j = 2 - 2 cos(j pi / (n+1)), j = 1..k."""
    n, k = 300, 8
    A = synth.laplacian_1d(n)
    negA = synth.CSR(A.n, A.row_ptr, A.col_idx, -A.val, name="negA")
    X0 = synth.gaussian_block(n, k + 1, 3)
    r = oracle.solve(negA, k, 10, 1, X0, tol=1e-10, w=k + 1)
    lam = 2 - 2 * np.cos(np.arange(1, k + 1) * np.pi / (n + 1))
    assert r.converged
    np.testing.assert_allclose(-r.mu, lam, rtol=1e-10)


def test_gn_step_fixed_point_and_solve():
    """Alg. GN: at X = V diag(sqrt(theta)) with V eigenvectors of the
    (filtered) operator, theta its eigenvalues > 0, X is a fixed point of
    X+ = Z - X (Y^T Z - I)/2 with Z = op(Y), Y = X (X^T X)^{-1}; and the GN inner
    solver inside the fixed-parameter driver converges to the closed-form spectrum."""
    n, k = 120, 6
    A = synth.laplacian_1d(n)
    lam = 2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))
    V = np.sqrt(2.0 / (n + 1)) * np.sin(np.outer(np.arange(1, n + 1), np.arange(1, n + 1)) * np.pi / (n + 1))
    a, b, d = 0.0, 3.2, 4
    theta = oracle.chebyshev_T(d, (lam - 1.6) / 1.6)  # rho_d on the spectrum
    top = np.argsort(theta)[::-1][:k]
    X = V[:, top] * np.sqrt(theta[top])
    Xp = oracle.gn_step(A, a, b, d, X)
    assert np.linalg.norm(Xp - X) <= 1e-10 * np.linalg.norm(X)
    X0 = synth.gaussian_block(300, k + 1, 2)
    r = oracle.solve(synth.laplacian_1d(300), k, 8, 1, X0, tol=1e-10, w=k + 1, inner_solver="gn")
    ref = (2 - 2 * np.cos(np.arange(1, 301) * np.pi / 301))[::-1][:k]
    assert r.converged and np.max(np.abs(r.mu - ref) / ref) < 1e-10
