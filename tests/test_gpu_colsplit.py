"""Column-partitioned multi-GPU mode (eig_init_colsplit; Survey §8f-3) on ONE GPU: G ranks
of an in-process communicator group, one host thread and stream per rank.  MPM filters
every column independently, so with A replicated the filter of a column slice
needs no exchange and its un-normalised output is bitwise the single-GPU filter's columns;
the ARR projection runs on the internal row partition after an all-to-all transpose, so its
Ritz values agree with one GPU to rounding (allreduce order) and solves converge to the same
eigenvalues within 1e-10."""
import numpy as np
import pytest
import torch

import oracle
import synth
from synth import configs

from test_gpu_dist import run_ranks

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def arr():
    import paper_1507_06078_b200 as m
    return m


CASES = {
    "zipf": lambda: synth.zipf_random(5000, 3),
    "lap3dV": lambda: synth.laplacian_3d_potential(13, 2),
    "lap2d": lambda: synth.laplacian_2d(40),
}


def make(arr, A, G, k, p, d, w, stencil=None):
    pt = arr.partition
    comms = arr.Comm.local_group(G)
    plans = [pt.colsplit_plan(A, w, G, r) for r in range(G)]

    def ctx_of(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            Af = arr.to_device_csr(A)
            Ar = arr.to_device_csr(plans[r].rows)
        s.synchronize()
        c = arr.eig_init_colsplit(Af, Ar, plans[r], k, p, d, w, comms[r], stream=s)
        if stencil:
            c.eig_set_stencil(*stencil)
        return c, s

    return plans, comms, ctx_of


@pytest.mark.parametrize("kind", list(CASES))
@pytest.mark.parametrize("G", [2, 3])
def test_colsplit_filter_is_local_and_bitwise(arr, kind, G):
    A = CASES[kind]()
    w, d = 36, 7
    X = synth.gaussian_block(A.n, w, 5)
    a = oracle.gershgorin_lower(A)
    b = a + 0.6 * (2 * np.abs(A.val).max() - a)
    one = arr.eig_init(arr.to_device_csr(A), w, 1, d, w=w)
    one.eig_set_interval(a, b)
    Xd = torch.from_numpy(X).cuda()
    one.filter_step(Xd, normalize=False)
    ref = Xd.cpu().numpy()
    plans, comms, ctx_of = make(arr, A, G, w, 1, d, w)

    def body(r):
        ctx, s = ctx_of(r)
        c0, c1 = plans[r].col_range
        with torch.cuda.stream(s):
            Xs = torch.from_numpy(np.ascontiguousarray(X[:, c0:c1])).cuda()
            ctx.eig_set_interval(a, b)
            l0 = ctx.launch_count
            ctx.filter_step(Xs, normalize=False)
            s.synchronize()
        out = (Xs.cpu().numpy(), ctx.launch_count - l0)
        ctx.close()
        return out

    res = run_ranks(G, body)
    for c in comms:
        c.close()
    for r in range(G):
        c0, c1 = plans[r].col_range
        assert np.array_equal(res[r][0], ref[:, c0:c1])


@pytest.mark.parametrize("kind", list(CASES))
def test_colsplit_arr_and_residuals(arr, kind):
    A = CASES[kind]()
    G, w, p = 2, 24, 2
    X = synth.gaussian_block(A.n, w, 9)
    a = oracle.gershgorin_lower(A)
    b = a + 0.7 * (2 * np.abs(A.val).max() - a)
    X = oracle.mpm_sweep(A, a, b, 4, X)
    one = arr.eig_init(arr.to_device_csr(A), w, p, 4, w=w)
    Yd = torch.zeros(A.n, w, dtype=torch.float64, device="cuda")
    ritz1, rank1 = one.arr_project(torch.from_numpy(X).cuda(), Yd)
    res1 = one.residuals(Yd, ritz1[:w])
    plans, comms, ctx_of = make(arr, A, G, w, p, 4, w)

    def body(r):
        ctx, s = ctx_of(r)
        c0, c1 = plans[r].col_range
        with torch.cuda.stream(s):
            Xs = torch.from_numpy(np.ascontiguousarray(X[:, c0:c1])).cuda()
            Ys = torch.zeros_like(Xs)
            ritz, rank = ctx.arr_project(Xs, Ys)
            res = ctx.residuals(Ys, ritz[:w])
            s.synchronize()
        out = (ritz, rank, res, Ys.cpu().numpy())
        ctx.close()
        return out

    out = run_ranks(G, body)
    for c in comms:
        c.close()
    scale = 2 * np.abs(A.val).max()
    for r in range(G):
        ritz, rank, res, _ = out[r]
        assert rank == rank1
        assert np.max(np.abs(ritz - ritz1)) <= 1e-12 * scale
        assert np.max(np.abs(res - res1)) <= 1e-10 * max(1.0, res1.max())
    # the Ritz vectors assembled from the column slices are orthonormal and match the oracle's residuals
    Y = np.hstack([out[r][3] for r in range(G)])
    assert np.linalg.norm(Y.T @ Y - np.eye(w)) < 1e-12
    ref = oracle.residuals(A, Y, out[0][0][:w])
    assert np.max(np.abs(ref - out[0][2])) <= 1e-10 * max(1.0, ref.max())


@pytest.mark.parametrize("kind,G", [("zipf", 2), ("lap3dV", 3), ("lap2d", 2)])
def test_colsplit_solve(arr, kind, G):
    spec = configs.SMALL_ANALOGS[kind]
    A, _ = configs.build_config(spec)
    X0 = configs.starting_block(spec)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    stencil = (spec.size, spec.size, spec.size) if kind == "lap3dV" else None
    plans, comms, ctx_of = make(arr, A, G, spec.k, spec.p, spec.d, spec.w, stencil=stencil)

    def body(r):
        ctx, s = ctx_of(r)
        c0, c1 = plans[r].col_range
        with torch.cuda.stream(s):
            Xs = torch.from_numpy(np.ascontiguousarray(X0[:, c0:c1])).cuda()
            ev, res, info = ctx.eig_solve(Xs, tol=spec.tol)
            s.synchronize()
        out = (ev, res, info.converged, info.outer, Xs.cpu().numpy())
        ctx.close()
        return out

    out = run_ranks(G, body)
    for c in comms:
        c.close()
    for r in range(G):
        ev, res, conv, outer, _ = out[r]
        assert conv and np.all(res <= spec.tol)
        assert np.max(np.abs(ev - lam) / np.abs(lam)) <= 1e-10
        assert np.array_equal(ev, out[0][0])  # identical on every rank
    # the k Ritz vectors assembled from the slices: the oracle's residual certificate
    Y = np.hstack([out[r][4] for r in range(G)])[:, :spec.k]
    cert = oracle.residuals(A, Y, out[0][0])
    assert np.all(cert <= 1.01 * spec.tol)
