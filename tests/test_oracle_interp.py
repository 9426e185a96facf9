"""Pins of the oracle's interpolant filter (the paper's default polynomial
accelerator, §5; R18): psi_d interpolates
f_d(t) = max(0,t)^{10d} at the Chebyshev points of the second kind, closed forms
for d = 1, 2, the paper's monomial form (Eq. chebfun-f) and Alg. poly's Horner
recurrence at small d, and rho_d(A) on diagonal A / by dense eigendecomposition."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("d", [1, 2, 3, 5, 10, 15, 20, 30])
def test_interpolates_f_d_at_second_kind_points(d):
    a = oracle.interp_coeffs(d)
    t = -np.cos(np.arange(d + 1) * np.pi / d)
    f = np.maximum(0.0, t) ** (10 * d)          # Eq. def:fN
    assert np.abs(oracle.psi(a, t) - f).max() <= 1e-14
    assert oracle.psi(a, np.array([1.0]))[0] == pytest.approx(1.0, abs=1e-14)  # f_d(1) = 1


def test_closed_forms_d1_d2():
    # d = 1: nodes -1, 1 with values 0, 1 -> psi_1(t) = (1 + t)/2 = T_0/2 + T_1/2
    np.testing.assert_allclose(oracle.interp_coeffs(1), [0.5, 0.5], atol=1e-16)
    # d = 2: nodes -1, 0, 1 with values 0, 0, 1 -> psi_2(t) = t(t+1)/2 = T_0/4 + T_1/2 + T_2/4
    np.testing.assert_allclose(oracle.interp_coeffs(2), [0.25, 0.5, 0.25], atol=1e-16)


@pytest.mark.parametrize("d", [3, 6, 10])
def test_monomial_form_and_alg_poly_agree_at_small_degree(d):
    """The paper's representation psi_d = gamma_1 t^d + ... + gamma_{d+1} (Eq.
    chebfun-f), from the Vandermonde system at the same nodes, and Alg. poly's
    Horner recurrence Y = c_0 Y + c_1 A Y + gamma_{j+1} X."""
    t = -np.cos(np.arange(d + 1) * np.pi / d)
    gamma = np.linalg.solve(np.vander(t, d + 1), np.maximum(0.0, t) ** (10 * d))
    a = oracle.interp_coeffs(d)
    s = np.linspace(-1.3, 1.3, 41)
    np.testing.assert_allclose(oracle.psi(a, s), np.polyval(gamma, s), rtol=1e-11, atol=1e-13)
    A = synth.laplacian_2d(9)
    X = synth.gaussian_block(A.n, 3, 4)
    lo, hi = 0.0, 6.0
    c0, c1 = (lo + hi) / (lo - hi), 2.0 / (hi - lo)
    Y = gamma[0] * X
    Ad = A.to_dense()
    for j in range(1, d + 1):  # Alg. poly, dense multiply
        Y = c0 * Y + c1 * (Ad @ Y) + gamma[j] * X
    Yo = oracle.poly_filter(A, lo, hi, a, X)
    assert np.linalg.norm(Yo - Y) / np.linalg.norm(Y) <= 1e-11


def test_rho_on_diagonal_matrix():
    dg = np.linspace(-2.0, 7.5, 60)
    A = synth.diagonal(dg)
    X = synth.gaussian_block(60, 4, 2)
    lo, hi, d = -2.0, 5.0, 12
    a = oracle.interp_coeffs(d)
    rho = oracle.psi(a, (2 * dg - lo - hi) / (hi - lo))  # Eq. rhod
    Y = oracle.poly_filter(A, lo, hi, a, X)
    np.testing.assert_allclose(Y, rho[:, None] * X, rtol=1e-12, atol=1e-14 * np.abs(rho).max())


def test_rho_by_dense_eigendecomposition():
    A = synth.zipf_random(200, 5)
    lam, Q = np.linalg.eigh(A.to_dense())
    X = synth.gaussian_block(200, 5, 6)
    lo, hi, d = float(lam[0]) - 0.1, float(np.quantile(lam, 0.8)), 10
    a = oracle.interp_coeffs(d)
    rho = oracle.psi(a, (2 * lam - lo - hi) / (hi - lo))
    ref = Q @ (rho[:, None] * (Q.T @ X))
    Y = oracle.poly_filter(A, lo, hi, a, X)
    assert np.linalg.norm(Y - ref) / np.linalg.norm(ref) <= 1e-11


def test_solve_with_interpolant_filter_small():
    spec = synth.SMALL_ANALOGS["lap2d"]
    A, _ = synth.build_config(spec)
    X0 = synth.starting_block(spec)
    r = oracle.solve(A, spec.k, spec.d, spec.p, X0, tol=spec.tol, filter="interp")
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    assert r.converged and np.max(np.abs(r.mu - lam) / lam) <= 1e-10
