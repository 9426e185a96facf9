"""Oracle pins: SpMM, Gershgorin bound, Chebyshev filter, MPM sweep.

Every expected value here comes from the paper's definitions worked by hand
(tests/golden), from closed forms of the operators, or from an independent
dense computation — never from the oracle itself.
"""
import os

import numpy as np
import pytest

import oracle
import synth
from synth.generators import from_dense

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rand_sym(n, seed, density=0.2):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
    a = a + a.T + np.diag(rng.standard_normal(n))
    return a


def _lap1d_eig(n):
    j = np.arange(1, n + 1)
    lam = 2 - 2 * np.cos(j * np.pi / (n + 1))
    x = np.arange(1, n + 1)
    V = np.sin(np.outer(x, j) * np.pi / (n + 1))
    return lam, V / np.linalg.norm(V, axis=0)


# ---------------------------------------------------------------- SpMM
def test_spmm_spec_trivial():
    A = synth.diagonal(np.array([1.0, 2.0, 3.0]))
    assert np.array_equal(oracle.spmm(A, np.ones((3, 1)))[:, 0], [1, 2, 3])
    Z = from_dense(np.zeros((4, 4)))
    assert np.array_equal(oracle.spmm(Z, np.ones((4, 2))), np.zeros((4, 2)))


def test_spmm_vs_dense_multiply():
    a = _rand_sym(60, 1)
    A = from_dense(a)
    X = np.random.default_rng(2).standard_normal((60, 7))
    Y = oracle.spmm(A, X)
    ref = a @ X
    assert np.linalg.norm(Y - ref) <= 1e-13 * np.linalg.norm(ref)
    # unit vectors give the dense columns exactly
    E = np.eye(60)
    assert np.max(np.abs(oracle.spmm(A, E) - a)) == 0


@pytest.mark.parametrize("build", [lambda: synth.laplacian_2d(11, 11), lambda: synth.stencil27_3d(7),
                                   lambda: synth.zipf_random(500, 9)])
def test_spmm_vs_dense_generators(build):
    A = build()
    X = np.random.default_rng(3).standard_normal((A.n, 5))
    ref = A.to_dense() @ X
    assert np.linalg.norm(oracle.spmm(A, X) - ref) <= 1e-13 * np.linalg.norm(ref)


def test_spmm_closed_form_eigenvectors():
    # 1-D: v_j(x) = sin(j pi x/(n+1)), lambda_j = 2 - 2cos(j pi/(n+1))
    n = 200
    lam, V = _lap1d_eig(n)
    A = synth.laplacian_1d(n)
    R = oracle.spmm(A, V) - V * lam
    assert np.max(np.abs(R)) < 1e-13
    # 27-point: A = 27 I - T(x)T(x)T, T = tridiag(1,1,1), eigvec = product of sines
    N = 6
    A = synth.stencil27_3d(N)
    x = np.arange(1, N + 1)
    for (i, j, k) in [(1, 1, 1), (2, 5, 3), (6, 6, 6)]:
        v = np.einsum("z,y,x->zyx", np.sin(k * np.pi * x / (N + 1)), np.sin(j * np.pi * x / (N + 1)),
                      np.sin(i * np.pi * x / (N + 1))).ravel()
        lam27 = 27 - np.prod([1 + 2 * np.cos(q * np.pi / (N + 1)) for q in (i, j, k)])
        r = oracle.spmm(A, v[:, None])[:, 0] - lam27 * v
        assert np.max(np.abs(r)) < 1e-12 * np.max(np.abs(v)) * 27


def test_spmm_symmetry_as_applied():
    A = synth.zipf_random(800, 4)
    rng = np.random.default_rng(5)
    X, Y = rng.standard_normal((800, 4)), rng.standard_normal((800, 3))
    lhs = Y.T @ oracle.spmm(A, X)
    rhs = oracle.spmm(A, Y).T @ X
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.abs(A.val).sum() / A.n * np.linalg.norm(X) * np.linalg.norm(Y)


# ---------------------------------------------------------------- Gershgorin
def test_gershgorin_lower():
    assert oracle.gershgorin_lower(synth.diagonal(np.array([1.0, 2.0, 3.0]))) == 1.0
    assert oracle.gershgorin_lower(from_dense(np.array([[2.0, 1.0], [1.0, 2.0]]))) == 1.0
    for A in (synth.laplacian_1d(50), synth.laplacian_2d(9), synth.stencil27_3d(5)):
        assert oracle.gershgorin_lower(A) == 0.0
    Z = synth.zipf_random(300, 1)  # diag = row abs-sum: 0 up to summation order
    assert abs(oracle.gershgorin_lower(Z)) <= 1e-13 * Z.val.max()
    A = synth.laplacian_3d_potential(6, 2)
    lo = oracle.gershgorin_lower(A)
    assert lo <= np.linalg.eigvalsh(A.to_dense()).min() + 1e-12
    a = _rand_sym(40, 7)
    assert oracle.gershgorin_lower(from_dense(a)) <= np.linalg.eigvalsh(a).min()


# ---------------------------------------------------------------- Chebyshev
def test_chebyshev_golden():
    rows = np.loadtxt(os.path.join(GOLD, "chebyshev_values.txt"))
    for d, t, v in rows:
        assert oracle.chebyshev_T(int(d), t) == pytest.approx(v, abs=1e-12)


def test_chebyshev_trig_closed_form():
    t = np.linspace(-1, 1, 101)
    for d in (1, 2, 7, 30):
        assert np.max(np.abs(oracle.chebyshev_T(d, t) - np.cos(d * np.arccos(t)))) < 1e-12
    t = np.array([1.01, 1.5, 3.0, -1.2, -2.5])
    for d in (3, 10, 30):
        ref = np.sign(t) ** d * np.cosh(d * np.arccosh(np.abs(t)))
        assert np.max(np.abs(oracle.chebyshev_T(d, t) / ref - 1)) < 1e-12


def _Td_closed(d, t):
    t = np.asarray(t, dtype=float)
    out = np.empty_like(t)
    m = np.abs(t) <= 1
    out[m] = np.cos(d * np.arccos(t[m]))
    out[~m] = np.sign(t[~m]) ** d * np.cosh(d * np.arccosh(np.abs(t[~m])))
    return out


@pytest.mark.parametrize("d", [0, 1, 2, 5, 10, 30])
def test_filter_diagonal_closed_form(d):
    rng = np.random.default_rng(d)
    diag = rng.uniform(-0.5, 4.0, 300)
    A = synth.diagonal(diag)
    a, b = 0.0, 3.0
    X = rng.standard_normal((300, 6))
    Y = oracle.cheb_filter(A, a, b, d, X)
    f = _Td_closed(d, (diag - 1.5) / 1.5)
    ref = f[:, None] * X
    assert np.linalg.norm(Y - ref) <= 1e-12 * np.linalg.norm(ref)


def test_filter_laplacian_eigenvectors():
    n, d, a, b = 300, 20, 0.0, 3.9
    lam, V = _lap1d_eig(n)
    A = synth.laplacian_1d(n)
    cols = [0, 1, 5, 150, 299]
    Y = oracle.cheb_filter(A, a, b, d, V[:, cols])
    ref = V[:, cols] * _Td_closed(d, (lam[cols] - 1.95) / 1.95)
    assert np.linalg.norm(Y - ref) <= 1e-12 * np.linalg.norm(ref)


def test_filter_degree_one_is_shifted_scaled_spmm():
    a = _rand_sym(50, 3)
    A = from_dense(a)
    X = np.random.default_rng(1).standard_normal((50, 4))
    Y = oracle.cheb_filter(A, -1.0, 2.0, 1, X)
    ref = (a @ X - 0.5 * X) / 1.5
    assert np.linalg.norm(Y - ref) <= 1e-13 * np.linalg.norm(ref)


def test_filter_bruteforce_dense_eig():
    # rho(A) = Q rho(Lambda) Q^T (Eq. poly-A), with numpy's eigh
    a = _rand_sym(150, 11, density=0.1)
    A = from_dense(a)
    lam, Q = np.linalg.eigh(a)
    lo, hi = lam.min() - 0.1, np.quantile(lam, 0.8)
    c, e = (lo + hi) / 2, (hi - lo) / 2
    X = np.random.default_rng(12).standard_normal((150, 5))
    for d in (3, 8, 15):
        ref = Q @ (_Td_closed(d, (lam - c) / e)[:, None] * (Q.T @ X))
        Y = oracle.cheb_filter(A, lo, hi, d, X)
        assert np.linalg.norm(Y - ref) <= 1e-11 * np.linalg.norm(ref)


def test_filter_column_subset_bitwise():
    A = synth.laplacian_2d(15)
    X = np.random.default_rng(4).standard_normal((A.n, 9))
    Y = oracle.cheb_filter(A, 0.0, 6.0, 12, X)
    cols = [0, 4, 8]
    Ys = oracle.cheb_filter(A, 0.0, 6.0, 12, X[:, cols])
    assert np.array_equal(Y[:, cols], Ys)


def test_filter_rejects_bad_interval():
    with pytest.raises(ValueError):
        oracle.cheb_filter(synth.laplacian_1d(10), 1.0, 1.0, 3, np.ones((10, 1)))


# ---------------------------------------------------------------- MPM
def test_mpm_spec_example():
    # A=diag(4,1), identity filter, X=[1;1]/sqrt2 -> [4;1]/sqrt(17).
    # T_1((t-c)/e) with [a,b]=[-1,1] is the identity map t -> t.
    A = synth.diagonal(np.array([4.0, 1.0]))
    X = np.array([[1.0], [1.0]]) / np.sqrt(2)
    Y = oracle.mpm_sweep(A, -1.0, 1.0, 1, X)
    assert np.allclose(Y[:, 0], np.array([4.0, 1.0]) / np.sqrt(17), rtol=0, atol=1e-15)


def test_mpm_unit_columns_and_column_norms():
    A = synth.laplacian_2d(12)
    X = np.random.default_rng(0).standard_normal((A.n, 6))
    Y = oracle.mpm_sweep(A, 0.0, 7.0, 8, X)
    assert np.max(np.abs(np.linalg.norm(Y, axis=0) - 1)) < 1e-14
    Z = np.random.default_rng(1).standard_normal((333, 4))
    assert np.allclose(oracle.col_norms(Z), np.sqrt((Z * Z).sum(0)), rtol=1e-14, atol=0)
