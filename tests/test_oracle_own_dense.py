"""Pins of the oracle's own dense steps (oracle/dense.py: pivoted and blocked
Householder QR, cyclic Jacobi, Cholesky, Gaussian elimination), the orthonormalise-
then-augment ARR variant (arr(method="cgs2"), R8) and the adaptive rules
of Alg. Arrabit2.  References: closed-form spectra and factorisations,
hand-computed rule decisions, and LAPACK (numpy / scipy) only as an independent
cross-check, never on the oracle path."""
import math

import numpy as np
import pytest
import scipy.linalg

import oracle
import synth
from oracle import dense
from synth import configs
from synth.generators import from_dense


def _rand_sym(n, seed):
    a = np.random.default_rng(seed).standard_normal((n, n))
    return a + a.T


# ------------------------------------------------------------------ QR
def test_qr_pivoted_factorises_and_pivots():
    rng = np.random.default_rng(1)
    Z = rng.standard_normal((200, 12)) * np.logspace(0, -6, 12)
    Q, R, piv = dense.qr_pivoted(Z)
    assert np.linalg.norm(Q.T @ Q - np.eye(12)) < 1e-14
    assert np.linalg.norm(Q @ R - Z[:, piv]) < 1e-14 * np.linalg.norm(Z)
    assert np.allclose(R, np.triu(R))
    d = np.abs(np.diag(R))
    assert np.all(d[:-1] >= d[1:] * (1 - 1e-12))  # pivoting orders |R_ii|
    # independent cross-check: LAPACK's pivoted QR has the same |R_ii|
    _, R2, _ = scipy.linalg.qr(Z, mode="economic", pivoting=True)
    assert np.allclose(d, np.abs(np.diag(R2)), rtol=1e-10)


def test_qr_pivoted_exact_rank():
    rng = np.random.default_rng(2)
    B = rng.standard_normal((150, 4))
    Z = B @ rng.standard_normal((4, 9))  # rank 4 exactly
    U, r = oracle.orthonormalize(Z)
    assert r == 4
    assert np.linalg.norm(Z - U @ (U.T @ Z)) < 1e-12 * np.linalg.norm(Z)


@pytest.mark.parametrize("m,nb", [(1, 32), (7, 3), (64, 32), (70, 32), (45, 8)])
def test_qr_blocked(m, nb):
    rng = np.random.default_rng(m)
    W = rng.standard_normal((300, m)) * np.logspace(0, -8, m)
    Q, R = dense.qr_blocked(W, nb=nb)
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) < 1e-14 * m
    assert np.linalg.norm(Q @ R - W) < 1e-14 * np.linalg.norm(W)
    assert np.allclose(R, np.triu(R))
    # unpivoted R agrees with LAPACK's up to the signs of the rows
    R2 = np.linalg.qr(W, mode="r")
    assert np.allclose(np.abs(R), np.abs(R2), atol=1e-12 * np.abs(R2).max())


def test_qr_blocked_rank_deficient_still_orthonormal():
    rng = np.random.default_rng(5)
    W = rng.standard_normal((200, 3)) @ rng.standard_normal((3, 20))
    Q, R = dense.qr_blocked(W, nb=8)
    assert np.linalg.norm(Q.T @ Q - np.eye(20)) < 1e-13
    assert np.linalg.norm(Q @ R - W) < 1e-13 * np.linalg.norm(W)


# ------------------------------------------------------------------ eig
def test_jacobi_closed_form_tridiagonal():
    m = 60
    T = 2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)
    lam, V = dense.jacobi_eigh(T)
    ref = np.sort(2 - 2 * np.cos(np.arange(1, m + 1) * np.pi / (m + 1)))
    assert np.max(np.abs(lam - ref)) < 2 * m * dense.EPS * 4  # backward error m eps ||T|| (Jacobi)
    assert np.linalg.norm(V.T @ V - np.eye(m)) < 1e-12
    assert np.linalg.norm(T @ V - V * lam) < 1e-12  # Frobenius over m columns


@pytest.mark.parametrize("m", [1, 2, 3, 17, 40])
def test_jacobi_random_vs_lapack(m):
    a = _rand_sym(m, m)
    lam, V = dense.jacobi_eigh(a)
    assert np.allclose(lam, np.linalg.eigvalsh(a), atol=1e-12 * max(1, np.abs(a).max()))
    assert np.linalg.norm(a @ V - V * lam) < 1e-12 * np.linalg.norm(a)
    assert np.all(np.diff(lam) >= 0)


def test_jacobi_multiple_eigenvalues():
    Q, _ = dense.qr_blocked(np.random.default_rng(3).standard_normal((12, 12)))
    d = np.array([5, 5, 5, 2, 2, 1, 0, 0, -1, -1, -1, -1], dtype=float)
    a = (Q * d) @ Q.T
    lam, V = dense.jacobi_eigh(a)
    assert np.allclose(lam, np.sort(d), atol=1e-13)
    assert np.linalg.norm(a @ V - V * lam) < 1e-13


# ------------------------------------------------------------------ small solves
def test_cholesky_and_triangular_solve():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((40, 9))
    G = X.T @ X
    R = dense.cholesky_upper(G)
    assert np.allclose(R, np.triu(R))
    assert np.linalg.norm(R.T @ R - G) < 1e-13 * np.linalg.norm(G)
    Qx = dense.solve_upper_right(X, R)  # X R^{-1} is orthonormal (Cholesky QR)
    assert np.linalg.norm(Qx.T @ Qx - np.eye(9)) < 1e-12
    with pytest.raises(FloatingPointError):
        dense.cholesky_upper(np.array([[1.0, 2.0], [2.0, 1.0]]))


def test_gepp_hand_and_pivoting():
    M = np.array([[0.0, 2.0, 1.0], [1.0, 1.0, 0.0], [2.0, 0.0, 3.0]])
    a = np.array([1.0, -2.0, 0.5])
    assert np.allclose(dense.solve_gepp(M, M @ a), a, atol=1e-15)  # needs a row swap (M_00 = 0)


# ------------------------------------------------------------------ cgs2 ARR variant
def test_arr_cgs2_equals_qr_on_closed_form():
    n, k = 300, 8
    A = synth.laplacian_1d(n)
    X = np.random.default_rng(7).standard_normal((n, k))
    for p in (0, 1, 2):
        mq, Yq, _ = oracle.arr(A, X, p, method="qr")
        mc, Yc, _ = oracle.arr(A, X, p, method="cgs2")
        m = (p + 1) * k
        assert np.allclose(mq[:m], mc[:m], rtol=0, atol=1e-13 * 4)
        assert np.linalg.norm(Yc.T @ Yc - np.eye(k)) < 1e-13
        # same Ritz subspace (cluster-free here): principal angles ~ 0
        s = np.linalg.svd(Yq.T @ Yc, compute_uv=False)
        assert s.min() > 1 - 1e-10


def test_arr_cgs2_exact_eigenvectors():
    n, k = 200, 6
    j = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(j * np.pi / (n + 1))
    V = np.sin(np.outer(j, j) * np.pi / (n + 1))
    V /= np.linalg.norm(V, axis=0)
    top = np.argsort(-lam)[:k]
    X = V[:, top] @ np.random.default_rng(2).standard_normal((k, k))
    mu, Y, _ = oracle.arr(synth.laplacian_1d(n), X, 2, method="cgs2")
    assert np.max(np.abs(mu[:k] - lam[top]) / lam[top]) < 1e-13
    assert np.max(oracle.residuals(synth.laplacian_1d(n), Y, mu[:k])) < 1e-12


def test_solve_cgs2_matches_closed_form():
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    N = spec.size
    c = 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    lam = np.sort((4 - c[:, None] - c[None, :]).ravel())[::-1]
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec), arr_method="cgs2")
    assert r.converged and np.all(r.res <= 1e-10)
    assert np.max(np.abs(r.mu - lam[:spec.k]) / lam[:spec.k]) < 1e-10


# ------------------------------------------------------------------ Alg. Arrabit2 rules
def test_rcond_gram_closed_form():
    rng = np.random.default_rng(8)
    U, _ = dense.qr_blocked(rng.standard_normal((100, 5)))
    W, _ = dense.qr_blocked(rng.standard_normal((5, 5)))
    s = np.array([3.0, 1.0, 0.5, 0.1, 0.01])
    X = (U * s) @ W.T
    assert oracle.rcond_gram(X) == pytest.approx((0.01 / 3.0) ** 2, rel=1e-10)


def test_degree_rule_hand_values():
    # a = 0, b = 1 -> c = e = 1/2; mu_k = 1.1 -> t = 1.2, mu_w = 1.05 -> t = 1.1
    # T_3(1.2) = 4(1.728) - 3(1.2) = 3.312, T_3(1.1) = 4(1.331) - 3.3 = 2.024: 0.611 < 0.9 -> d = 3
    assert oracle.core._degree_rule(15, 0.0, 1.0, 1.1, 1.05) == 3
    # mu_w very close to mu_k: the ratio only falls below 0.9 at a higher degree
    t_k, t_w = 1.0 + 2e-3, 1.0 + 1e-3
    mu_k, mu_w = 0.5 + 0.5 * t_k, 0.5 + 0.5 * t_w
    d = next(dd for dd in range(3, 200)
             if abs(oracle.chebyshev_T(dd, t_w)) < 0.9 * abs(oracle.chebyshev_T(dd, t_k)))
    assert d > 3
    assert oracle.core._degree_rule(200, 0.0, 1.0, mu_k, mu_w) == d
    assert oracle.core._degree_rule(d - 1, 0.0, 1.0, mu_k, mu_w) == d - 1  # cap d_max (Eq. degree)


def test_continuation_and_deflation_rules():
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    N = spec.size
    c = 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    lam = np.sort((4 - c[:, None] - c[None, :]).ravel())[::-1]
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec), adapt=4)
    assert r.converged and np.max(np.abs(r.mu - lam[:spec.k]) / lam[:spec.k]) < 1e-10
    tols = [e["tol_t"] for e in r.log]
    assert tols[0] == pytest.approx(math.sqrt(1e-10))
    for t0, t1 in zip(tols, tols[1:]):  # Eq. contin: tol_{t+1} in {tol_t, max(1e-2 tol_t, tol)}
        assert t1 == t0 or t1 == pytest.approx(max(1e-2 * t0, 1e-10))
    locked = [e["locked"] for e in r.log]
    assert locked == sorted(locked)  # locked pairs never come back
    with pytest.raises(ValueError):
        oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec), adapt=5)


def test_adaptive_p_and_d_rules_converge():
    spec = configs.SMALL_ANALOGS["lap3dV"]
    A, _ = configs.build_config(spec)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec), adapt=3)
    assert r.converged and np.max(np.abs(r.mu - lam) / lam) < 1e-10
    ps = [e["p"] for e in r.log]
    ds = [e["d"] for e in r.log]
    assert ps[0] == 1 and ps == sorted(ps) and max(ps) <= spec.p  # Eq. block only increases p
    assert ds[0] == 3 and all(3 <= x <= spec.d for x in ds)
    # each recorded degree is the rule's choice from the most accurate Ritz pair so far
    # (checked in the GPU comparison test against the same oracle run)


def test_rcond_inner_rule_and_exits():
    spec = configs.SMALL_ANALOGS["lap2d"]
    A, _ = configs.build_config(spec)
    r = oracle.solve(A, spec.k, spec.d, spec.p, synth.starting_block(spec), inner="rcond", exits=3)
    assert all(e["s"] % 5 == 0 and 5 <= e["s"] <= 50 for e in r.log)
    assert r.exit_rule in (1, 2, 3)
    if r.exit_rule == 3:  # (iii): max res < (1 + 9h/k) tol
        assert r.res.max() < 10 * 1e-10


def test_ritz_lapack_switch_equals_jacobi():
    """oracle.core.EIGH = "lapack" (the cfg3 golden's m = 1650 projected problems,
    scripts/oracle_golden.py --eigh lapack) gives the Ritz values and the Ritz subspaces of
    the default cyclic Jacobi (Alg. RR step 3)."""
    import oracle.core as oc
    import synth
    A = synth.laplacian_3d_potential(7, 2)
    X = synth.gaussian_block(A.n, 12, 3)
    assert oc.EIGH == "jacobi"
    mu_j, Y_j, r_j = oc.arr(A, X, 2, method="cgs2")
    try:
        oc.EIGH = "lapack"
        mu_l, Y_l, r_l = oc.arr(A, X, 2, method="cgs2")
    finally:
        oc.EIGH = "jacobi"
    assert r_j == r_l
    assert np.max(np.abs(mu_j - mu_l)) <= 1e-13 * np.max(np.abs(mu_j))
    # same residuals of the kept pairs (vectors agree up to sign / rotations inside clusters)
    rj = oc.residuals(A, Y_j, mu_j[:12])
    rl = oc.residuals(A, Y_l, mu_l[:12])
    assert np.max(np.abs(rj - rl)) <= 1e-12
