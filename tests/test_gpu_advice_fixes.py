"""Regression tests for the round-1 advisor findings:
GN's Cholesky info is checked (a singular X^T X fails loudly), unsupported option
combinations with continuation + deflation are rejected, gram() refuses products larger
than the partial-sum buffer, p is bounded, and spmm() on a distributed context runs the
halo exchange (bitwise the single-GPU product on the owned rows)."""
import numpy as np
import pytest
import torch

import synth

from test_gpu_dist import make_rank, run_ranks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def arr():
    import paper_1507_06078_b200 as m
    return m


def test_gn_singular_gram_fails_loudly(arr):
    A = synth.laplacian_2d(30)
    X = synth.gaussian_block(A.n, 10, 1)
    X[:, 7] = X[:, 3]  # X^T X singular
    ctx = arr.eig_init(arr.to_device_csr(A), 10, 1, 4)
    with pytest.raises(arr.ArrError) as e:
        ctx.eig_solve(torch.from_numpy(X).cuda(), tol=1e-10, maxit=2, inner_solver="gn")
    assert e.value.status == 7  # ARR_ENUMERIC


@pytest.mark.parametrize("opt", [dict(adapt=5), dict(adapt=6), dict(adapt=4, inner="rcond"), dict(adapt=4, exits=1),
                                 dict(adapt=4, inner_solver="gn")])
def test_deflation_rejects_unsupported_combinations(arr, opt):
    A = synth.laplacian_2d(30)
    ctx = arr.eig_init(arr.to_device_csr(A), 8, 1, 4)
    with pytest.raises(arr.ArrError) as e:
        ctx.eig_solve(torch.from_numpy(synth.gaussian_block(A.n, 8, 2)).cuda(), tol=1e-10, maxit=2, **opt)
    assert e.value.status == 1  # ARR_EINVAL


def test_gram_larger_than_partials_is_rejected(arr):
    n = 3000
    ctx = arr.eig_init(arr.to_device_csr(synth.laplacian_1d(n)), 20, 1, 3)
    X = torch.randn(n, 3000, dtype=torch.float64, device="cuda")
    G = torch.empty(3000, 3000, dtype=torch.float64, device="cuda")
    with pytest.raises(arr.ArrError) as e:
        ctx.gram(X, X, G)
    assert e.value.status == 1


def test_p_bound(arr):
    A = synth.laplacian_1d(5000)
    with pytest.raises(arr.ArrError):
        arr.eig_init(arr.to_device_csr(A), 4, 17, 3)
    arr.eig_init(arr.to_device_csr(A), 4, 16, 3).close()


def test_spmm_on_distributed_context_exchanges_halo(arr):
    A = synth.laplacian_3d_potential(12, 2)
    G, w = 2, 10
    X = synth.gaussian_block(A.n, w, 3)
    one = arr.eig_init(arr.to_device_csr(A), w, 1, 3)
    Y1 = torch.zeros(A.n, w, dtype=torch.float64, device="cuda")
    one.spmm(torch.from_numpy(X).cuda(), Y1, alpha=0.5, shift=1.5)
    ref = Y1.cpu().numpy()
    ps, comms, ctx_of = make_rank(arr, A, G, ("planes", 12, 144), w, 1, 3)

    def body(r):
        ctx, s = ctx_of(r)
        p = ps[r]
        with torch.cuda.stream(s):
            Xl = torch.zeros(p.n_rows_block, w, dtype=torch.float64, device="cuda")
            Xl[:p.n_own] = torch.from_numpy(X[p.row_begin:p.row_begin + p.n_own]).cuda()  # ghost rows left zero
            Yl = torch.zeros_like(Xl)
            ctx.spmm(Xl, Yl, alpha=0.5, shift=1.5)
            s.synchronize()
        out = Yl[:p.n_own].cpu().numpy()
        ctx.close()
        return out

    out = run_ranks(G, body)
    for c in comms:
        c.close()
    for r in range(G):
        p = ps[r]
        assert np.array_equal(out[r], ref[p.row_begin:p.row_begin + p.n_own])
