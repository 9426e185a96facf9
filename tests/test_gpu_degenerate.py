"""Degenerate and boundary inputs of the hot path against the oracle / closed forms:
empty CSR rows, a single column (w = 1), degree 1, no augmentation (p = 0), the smallest n
the ARR allows ((p+1)w = n - 1, Alg. ARR input P:536), the zero matrix (every eigenvalue 0:
the interval safeguard of R3 makes a < b), and a diagonal matrix whose top eigenvalue is
repeated (a cluster across the k-th pair, R9)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth.generators import CSR

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def arr():
    import paper_1507_06078_b200 as m
    return m


def _with_empty_rows(n, seed):
    """A symmetric tridiagonal-plus-diagonal matrix in which every 7th row (and column)
    is empty."""
    rng = np.random.default_rng(seed)
    dense = np.diag(rng.uniform(1, 3, n))
    for i in range(n - 1):
        dense[i, i + 1] = dense[i + 1, i] = rng.uniform(-1, 1)
    dead = np.arange(0, n, 7)
    dense[dead, :] = 0
    dense[:, dead] = 0
    return synth.generators.from_dense(dense), dense


@pytest.mark.parametrize("w", [1, 2, 9])
def test_empty_rows_spmm_filter_and_arr(arr, w):
    A, dense = _with_empty_rows(300, 1)
    assert np.any(np.diff(A.row_ptr) == 0)
    X = synth.gaussian_block(A.n, w, 2)
    ctx = arr.eig_init(arr.to_device_csr(A), w, 1, 5)
    Yd = torch.zeros(A.n, w, dtype=torch.float64, device="cuda")
    ctx.spmm(torch.from_numpy(X).cuda(), Yd, alpha=1.0, shift=0.25)
    ref = dense @ X - 0.25 * X
    assert np.linalg.norm(Yd.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    a = oracle.gershgorin_lower(A)
    ctx.eig_set_interval(a, a + 2.0)
    Xd = torch.from_numpy(X).cuda()
    ctx.filter_step(Xd, normalize=False)
    Y = oracle.cheb_filter(A, a, a + 2.0, 5, X)
    assert np.linalg.norm(Xd.cpu().numpy() - Y) <= 1e-12 * np.linalg.norm(Y)


def test_single_column_degree_one_p0(arr):
    A = synth.laplacian_2d(20)
    X = synth.gaussian_block(A.n, 1, 3)
    ctx = arr.eig_init(arr.to_device_csr(A), 1, 0, 1)
    ctx.eig_set_interval(0.0, 4.0)
    Xd = torch.from_numpy(X).cuda()
    ctx.filter_step(Xd, normalize=False)
    ref = (oracle.spmm(A, X) - 2.0 * X) / 2.0  # d = 1: (A - cI) X / e
    assert np.linalg.norm(Xd.cpu().numpy() - ref) <= 1e-13 * np.linalg.norm(ref)
    Yd = torch.zeros_like(Xd)
    ritz, rank = ctx.arr_project(Xd, Yd, p=0)
    y = Xd.cpu().numpy()[:, 0]
    assert rank == 1 and ritz[0] == pytest.approx(y @ oracle.spmm(A, y) / (y @ y), rel=1e-13)


def test_smallest_n_for_arr(arr):
    k, p = 6, 2
    n = (p + 1) * k + 1
    A = synth.laplacian_1d(n)
    lam = np.sort(2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)))[::-1]
    ctx = arr.eig_init(arr.to_device_csr(A), k, p, 4)
    ev, res, info = ctx.eig_solve(torch.from_numpy(synth.gaussian_block(n, k, 4)).cuda(), tol=1e-10)
    assert info.converged and np.max(np.abs(ev - lam[:k]) / lam[:k]) <= 1e-10
    with pytest.raises(arr.ArrError):
        arr.eig_init(arr.to_device_csr(A), k + 1, p, 4)  # (p+1) w >= n


def test_zero_matrix(arr):
    n, k = 200, 4
    A = CSR(n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int32), np.zeros(0), "zero")
    ctx = arr.eig_init(arr.to_device_csr(A), k, 1, 3)
    assert ctx.eig_gershgorin_lower() == 0.0
    ev, res, info = ctx.eig_solve(torch.from_numpy(synth.gaussian_block(n, k, 5)).cuda(), tol=1e-10, maxit=5)
    assert info.converged and np.all(ev == 0.0) and np.all(res == 0.0)


def test_repeated_top_eigenvalue(arr):
    n, k = 400, 5
    d = np.linspace(1.0, 2.0, n)
    d[-3:] = 3.0  # lambda_1 = lambda_2 = lambda_3 = 3
    A = synth.generators.diagonal(d)
    lam = np.sort(d)[::-1][:k]
    ctx = arr.eig_init(arr.to_device_csr(A), k, 1, 6, w=k + 2)
    X0 = synth.gaussian_block(n, k + 2, 6)
    ev, res, info = ctx.eig_solve(torch.from_numpy(X0).cuda(), tol=1e-10)
    assert info.converged and np.max(np.abs(ev - lam) / lam) <= 1e-10
    ro = oracle.solve(A, k, 6, 1, X0, tol=1e-10)
    assert np.max(np.abs(ro.mu - ev) / lam) <= 1e-10
