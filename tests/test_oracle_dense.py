"""Oracle pins: orthonormalisation, RR, ARR, residuals (Alg. RR P:213-226,
Alg. ARR, Eq. resi).  References are closed-form spectra,
exact invariant subspaces, and an independent orthonormalisation (SVD) +
numpy eigvalsh."""
import numpy as np
import pytest

import oracle
import synth
from synth.generators import from_dense


def _rand_sym(n, seed):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n))
    return a + a.T


def _lap1d_eig(n):
    j = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(j * np.pi / (n + 1))
    x = np.arange(1, n + 1)
    V = np.sin(np.outer(x, j) * np.pi / (n + 1))
    return lam, V / np.linalg.norm(V, axis=0)


def test_orthonormalize_spec_examples():
    Z = 2 * np.eye(6)[:, :3]
    U, r = oracle.orthonormalize(Z)
    assert r == 3 and np.allclose(np.abs(U), np.eye(6)[:, :3], atol=1e-15)
    rng = np.random.default_rng(0)
    Z = rng.standard_normal((100, 10))
    Z[:, 7] = Z[:, 2]
    U, r = oracle.orthonormalize(Z)
    assert r == 9
    assert np.linalg.norm(U.T @ U - np.eye(9)) < 1e-13
    assert np.linalg.norm(Z - U @ (U.T @ Z)) < 1e-12 * np.linalg.norm(Z)


def test_rr_invariant_subspace_diag():
    A = synth.diagonal(np.array([3.0, 2.0, 1.0]))
    mu, Y, r = oracle.rayleigh_ritz(A, np.eye(3)[:, :2])
    assert r == 2 and np.allclose(mu, [3, 2], atol=1e-15)
    assert np.max(oracle.residuals(A, Y, mu)) < 1e-15


def test_rr_full_space_is_dense_eig():
    a = _rand_sym(30, 3)
    mu, Y, r = oracle.rayleigh_ritz(from_dense(a), np.eye(30))
    assert r == 30
    assert np.allclose(mu, np.sort(np.linalg.eigvalsh(a))[::-1], atol=1e-12)
    assert np.linalg.norm(Y.T @ Y - np.eye(30)) < 1e-12


def test_arr_exact_eigenvectors_lap1d():
    n, k = 400, 10
    lam, V = _lap1d_eig(n)
    A = synth.laplacian_1d(n)
    top = np.argsort(-lam)[:k]
    X = V[:, top] @ np.random.default_rng(1).standard_normal((k, k))  # same span, mixed
    for p in (0, 1, 2):
        mu, Y, r = oracle.arr(A, X, p)
        assert np.max(np.abs(mu[:k] - lam[top]) / lam[top]) < 1e-13
        assert np.max(oracle.residuals(A, Y, mu[:k])) < 1e-12


def test_arr_p0_equals_rr():
    A = synth.zipf_random(400, 2)
    X = np.random.default_rng(3).standard_normal((400, 8))
    mu0, Y0, _ = oracle.arr(A, X, 0)
    mu1, Y1, _ = oracle.rayleigh_ritz(A, X)
    assert np.array_equal(mu0, mu1)
    assert np.array_equal(Y0, Y1[:, :8])


def test_arr_vs_independent_projection():
    # RR on span{X, AX, A^2X}: an SVD-based basis (independent of pivoted QR)
    a = _rand_sym(60, 5)
    A = from_dense(a)
    X = np.random.default_rng(6).standard_normal((60, 5))
    Z = np.hstack([X, a @ X, a @ (a @ X)])
    Uz, s, _ = np.linalg.svd(Z / np.linalg.norm(Z, axis=0), full_matrices=False)
    B = Uz[:, s > 1e-10 * s[0]]
    ref = np.sort(np.linalg.eigvalsh(B.T @ a @ B))[::-1]
    mu, Y, r = oracle.arr(A, X, 2)
    assert r == B.shape[1] == 15
    assert np.allclose(mu, ref, rtol=0, atol=1e-11 * np.abs(ref).max())
    lam = np.sort(np.linalg.eigvalsh(a))[::-1]
    # Cauchy interlacing: mu_i <= lambda_i and mu_{m-i} >= lambda_{n-i}
    assert np.all(mu <= lam[:15] + 1e-12)
    assert np.all(mu[::-1] >= lam[::-1][:15] - 1e-12)
    assert np.linalg.norm(Y.T @ Y - np.eye(5)) < 1e-12
    # Ritz vectors satisfy the Galerkin condition B^T (A y - mu y) = 0
    R = a @ Y - Y * mu[:5]
    assert np.linalg.norm(B.T @ R) < 1e-10 * np.abs(ref).max()


def test_residuals_hand_example():
    A = synth.diagonal(np.array([3.0, 2.0, 1.0]))
    Y = np.array([[1.0], [0.0], [0.0]])
    # ||A e1 - 2.5 e1|| / max(1, 2.5) = 0.5 / 2.5
    assert oracle.residuals(A, Y, np.array([2.5]))[0] == pytest.approx(0.2, rel=1e-15)
    # |mu| < 1 uses the denominator 1
    assert oracle.residuals(A, Y, np.array([0.5]))[0] == pytest.approx(2.5, rel=1e-15)


def test_arr_beats_rr_on_flat_spectrum():
    # Thm thm:ARR1/Cor. and Table 2's claim: after the
    # same filtering, the k-th Ritz residual from ARR(p=1) is smaller than RR(p=0).
    n, k = 400, 20
    lam = 1 - 0.0005 * np.arange(n)
    Q, _ = np.linalg.qr(np.random.default_rng(0).standard_normal((n, n)))
    a = (Q * lam) @ Q.T
    a = 0.5 * (a + a.T)
    A = from_dense(a)
    wins = 0
    for seed in range(8):
        X = np.random.default_rng(100 + seed).standard_normal((n, k))
        X = oracle.mpm_sweep(A, 0.75, 0.99, 6, X)
        mu0, Y0, _ = oracle.arr(A, X, 0)
        mu1, Y1, _ = oracle.arr(A, X, 1)
        r0 = oracle.residuals(A, Y0, mu0[:k]).max()
        r1 = oracle.residuals(A, Y1, mu1[:k]).max()
        wins += r1 < r0
        # optimality: the partial trace from the larger space is never smaller
        assert mu1[:k].sum() >= mu0[:k].sum() - 1e-12
    assert wins == 8


def test_sweeps_rule():
    # amp <= 1 -> s_max; else floor(D / log10 amp) clamped to [1, s_max]: the thresholds of
    # amp for s = 1, 2, 3 sit at 10^D, 10^(D/2), 10^(D/3) (D = 12 default, D = 8 the round-1 value)
    assert oracle.RANGE_DIGITS == 12.0
    assert oracle.sweeps_rule(0.5, 0.0, 1.0, 10, 5) == 5
    d = 1  # T_1(t) = t: mu1 = amp * e + c gives (mu1 - c)/e = amp with c = e = 0.5
    for D in (8.0, 12.0):
        kw = {} if D == 12.0 else {"digits": D}
        assert oracle.sweeps_rule(10 ** (D + 1e-9) * 0.5 + 0.5, 0.0, 1.0, d, 5, **kw) == 1
        assert oracle.sweeps_rule(10 ** (D / 2 - 1e-6) * 0.5 + 0.5, 0.0, 1.0, d, 5, **kw) == 2
        assert oracle.sweeps_rule(10 ** (D / 3.0 + 1e-9) * 0.5 + 0.5, 0.0, 1.0, d, 5, **kw) == 2
        assert oracle.sweeps_rule(10 ** (D / 3.0 - 1e-6) * 0.5 + 0.5, 0.0, 1.0, d, 5, **kw) == 3
        assert oracle.sweeps_rule(10 ** (D / 7.0) * 0.5 + 0.5, 0.0, 1.0, d, 5, **kw) == 5  # capped at s_max
