"""GPU parity at BASELINE.json's FULL sizes (cfg3, cfg4, cfg5), in the launch
configuration of a solve (full block width w = k + q, the config's degree d).

* filter_step on the whole n x w block vs the oracle on a seeded sample of 16
  columns (exact, not approximate: p_d(A) acts on every column independently,
  P:555-566; SURVEY.md §8c-6 "column-sampled filter");
* cfg3: a full solve to tol = 1e-10, pinned by the oracle's own residual
  recomputation of every returned pair (Eq. resi) and by Weyl's
  bounds lambda_i(L) <= mu_i <= lambda_i(L) + max V with the closed-form 7-point
  Laplacian spectrum.
Inputs come from synth (seeded), uploaded in row chunks."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import configs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

CHUNK = 1 << 21


@pytest.fixture(scope="module")
def arr():
    import paper_1507_06078_b200 as m
    return m


def upload_X0(spec, n, cols):
    """X0 (n x w, stream 0 then q guard columns from stream 2) straight to the
    device in row chunks; returns (device block, host copy of the sampled columns)."""
    w = spec.w
    Xd = torch.empty((n, w), dtype=torch.float64, device="cuda")
    Xs = np.empty((n, len(cols)))
    for r0 in range(0, n, CHUNK):
        r1 = min(n, r0 + CHUNK)
        blk = synth.gaussian_block_rows(n, spec.k, spec.seed, r0, r1)
        if spec.q:
            blk = np.hstack([blk, synth.gaussian_block_rows(n, spec.q, spec.seed, r0, r1, stream=2)])
        Xd[r0:r1] = torch.from_numpy(blk)
        Xs[r0:r1] = blk[:, cols]
    return Xd, Xs


def gersh_upper(A):
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    return float(np.bincount(rows, weights=np.abs(A.val), minlength=A.n).max())


@pytest.mark.parametrize("cid", [3, 4, 5])
def test_fullsize_filter_step_sampled_columns(arr, cid):
    A, spec = configs.build_config(cid)
    cols = np.sort(np.random.default_rng(1234 + cid).choice(spec.w, 16, replace=False))
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, 0, spec.d, w=spec.w)
    a = ctx.eig_gershgorin_lower()
    assert a == oracle.gershgorin_lower(A)
    b = a + 0.9 * (gersh_upper(A) - a)
    ctx.eig_set_interval(a, b)
    Xd, Xs = upload_X0(spec, A.n, cols)
    nrm = torch.empty(spec.w, dtype=torch.float64, device="cuda")
    ctx.filter_step(Xd, normalize=True, colnorm=nrm)
    got = Xd[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    got_nrm = nrm.cpu().numpy()[cols]
    del Xd
    ctx.close()
    Y = oracle.cheb_filter(A, a, b, spec.d, Xs)
    ref_nrm = oracle.col_norms(Y)
    assert np.max(np.abs(got_nrm - ref_nrm) / ref_nrm) <= 1e-12
    ref = Y / ref_nrm
    err = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, err
    # unnormalised (rescaled by the GPU's own norms): the filter itself
    err_raw = np.linalg.norm(got * got_nrm - Y) / np.linalg.norm(Y)
    assert err_raw <= 1e-12, err_raw


def _lap3d_top(N, k):
    lam1 = 2 - 2 * np.cos(np.arange(1, N + 1) * np.pi / (N + 1))
    top = np.sort(lam1)[::-1][:k]  # the k largest sums use only the k largest 1-D values per axis
    s = (top[:, None, None] + top[None, :, None] + top[None, None, :]).ravel()
    return np.sort(s)[::-1][:k]


def test_fullsize_cfg3_solve_certified(arr):
    A, spec = configs.build_config(3)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd, _ = upload_X0(spec, A.n, [0])
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max)
    assert info.converged == 1 and np.all(res <= spec.tol)
    Y = Xd[:, :spec.k].cpu().numpy()
    del Xd
    ctx.close()
    cert = oracle.residuals(A, Y, ev)
    assert np.all(cert <= 1.01 * spec.tol)
    # Weyl with the closed-form Laplacian spectrum (lambda_1(L) = 11.99709769375193)
    lamL = _lap3d_top(100, spec.k)
    assert lamL[0] == pytest.approx(11.99709769375193, rel=1e-14)
    V = synth.generators.potential_uniform(A.n, spec.seed)
    assert np.all(ev >= lamL - 1e-9) and np.all(ev <= lamL + V.max() + 1e-9)
    # orthonormal Ritz vectors
    G = Y.T @ Y
    assert np.abs(G - np.eye(spec.k)).max() <= 1e-10


def test_fullsize_cfg4_solve_certified(arr):
    """cfg4 (random Zipf rows, n = 4e6, k = 1000) at full size: the solve converges
    and the oracle recomputes every returned pair's residual with its own SpMM
    (Eq. resi; full-scale cfg4 parity is residual
    certificates + the reduced-n oracle solve of tests/test_gpu_parity.py)."""
    A, spec = configs.build_config(4)
    ctx = arr.eig_init(arr.to_device_csr(A), spec.k, spec.p, spec.d, w=spec.w)
    Xd, _ = upload_X0(spec, A.n, [0])
    ev, res, info = ctx.eig_solve(Xd, tol=spec.tol, maxit=60, s_max=spec.s_max)
    assert info.converged == 1 and np.all(res <= spec.tol)
    Y = Xd[:, :spec.k].cpu().numpy()
    del Xd
    ctx.close()
    cert = oracle.residuals(A, Y, ev)
    assert np.all(cert <= 1.01 * spec.tol)
    assert np.all(np.diff(ev) <= 0)  # descending
    # Gershgorin: every eigenvalue of A lies in [a, max_i sum_j |A_ij|]
    assert ev[0] <= gersh_upper(A) and ev[-1] >= oracle.gershgorin_lower(A)
    G = Y.T @ Y
    assert np.abs(G - np.eye(spec.k)).max() <= 1e-10
