"""GPU parity of the distributed path (eig_init_dist)
on ONE GPU: G ranks of an in-process communicator group (comm_init_local_group),
one host thread and one stream per rank, each with its row block of A (local
CSR + ghost columns from partition.py).  The exchange, Gram allreduce and
broadcasts go through the same library code paths as NCCL, with device copies
instead of NCCL transfers.  Expected (§8(e) "Parity across G"): the
un-normalised filter is bitwise identical to one GPU; normalised blocks, Gram
products and Ritz values agree to rounding (allreduce order); solves converge
to the same eigenvalues within 1e-10."""
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from synth import configs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def arr():
    import paper_1507_06078_b200 as m
    return m


CASES = {
    "lap3dV": (lambda: synth.laplacian_3d_potential(13, 2), lambda G: ("planes", 13, 169)),
    "zipf": (lambda: synth.zipf_random(5000, 3), lambda G: ("balanced",)),
    "st27": (lambda: synth.stencil27_3d(11), lambda G: ("planes", 11, 121)),
    "lap2d": (lambda: synth.laplacian_2d(40), lambda G: ("planes", 40, 40)),
}


def _bounds(pt, A, spec, G):
    if spec[0] == "planes":
        return pt.bounds_planes(spec[1], spec[2], G)
    return pt.bounds_balanced(A.row_ptr, G)


def run_ranks(G, fn):
    """Run fn(rank) on G threads; return the list of results (re-raise the first error)."""
    out, err = [None] * G, [None] * G

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for e in err:
        if e is not None:
            raise e
    return out


def make_rank(arr, A, G, spec, k, p, d, w=None, yband=None):
    """Plans, communicators and a per-rank factory of (ctx, plan, stream)."""
    pt = arr.partition
    ps = pt.plans(A, _bounds(pt, A, spec, G), yband=yband)
    comms = arr.Comm.local_group(G)

    def ctx_of(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            Ad = arr.to_device_csr(ps[r])
        s.synchronize()
        return arr.eig_init(Ad, k, p, d, stream=s, w=w, comm=comms[r], plan=ps[r]), s

    return ps, comms, ctx_of


def to_rank_block(X, plan, ld=None):
    from paper_1507_06078_b200 import partition as pt
    blk = torch.from_numpy(pt.scatter_rows(X, plan, ld)).cuda()
    return blk[:, :X.shape[1]]


@pytest.mark.parametrize("kind,G,yb", [("lap3dV", 2, None), ("lap3dV", 3, None), ("zipf", 2, None), ("zipf", 3, None),
                                       ("st27", 4, None), ("lap2d", 2, None), ("lap3dV", 2, (13, 13, 4)),
                                       ("st27", 3, (11, 11, 3))])
def test_dist_filter_bitwise_and_normalised(arr, kind, G, yb):
    """yb: the interior tiles in y-band order (partition.local_plan(yband=...), bench.py's
    N > 1 default on the 3-D grids): the row order moves, the sums do not."""
    mk, sp = CASES[kind]
    A = mk()
    k, d = 24, 9
    X0 = synth.gaussian_block(A.n, k, 5)
    a = oracle.gershgorin_lower(A)
    b = a + 0.55 * (2 * float(np.abs(A.val).sum() / A.n * 2) - a)
    # single GPU reference (same kernels, no partition)
    c1 = arr.eig_init(arr.to_device_csr(A), k, 1, d)
    c1.eig_set_interval(a, b)
    X1 = torch.from_numpy(X0).cuda()
    c1.filter_step(X1, normalize=False)
    ref_raw = X1.cpu().numpy()
    X1 = torch.from_numpy(X0).cuda()
    c1.filter_step(X1, normalize=True)
    ref_nrm = X1.cpu().numpy()
    ps, comms, ctx_of = make_rank(arr, A, G, sp(G), k, 1, d, yband=yb)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            ctx.eig_set_interval(a, b)
            Xr = to_rank_block(X0, ps[r])
            ctx.filter_step(Xr, normalize=False)
            raw = Xr[:ps[r].n_own].cpu().numpy()
            Xr = to_rank_block(X0, ps[r], ld=k + 2)  # padded ld: packed-exchange path
            ctx.filter_step(Xr, normalize=True)
            nrm = Xr[:ps[r].n_own].cpu().numpy()
        ctx.close()
        return raw, nrm

    res = run_ranks(G, work)
    for c in comms:
        c.close()
    raw = np.vstack([x[0] for x in res])
    nrm = np.vstack([x[1] for x in res])
    assert np.array_equal(raw, ref_raw), "un-normalised distributed filter is not bitwise equal"
    assert np.abs(nrm - ref_nrm).max() <= 1e-14
    orc = oracle.mpm_sweep(A, a, b, d, X0)
    assert np.linalg.norm(nrm - orc) / np.linalg.norm(orc) <= 1e-12


@pytest.mark.parametrize("kind,G,p", [("lap3dV", 3, 2), ("zipf", 2, 1), ("st27", 2, 2)])
def test_dist_arr_gram_residuals(arr, kind, G, p):
    mk, sp = CASES[kind]
    A = mk()
    k = 16
    X0 = synth.gaussian_block(A.n, k, 9)
    mu_o, _, _ = oracle.arr(A, X0, p)
    ps, comms, ctx_of = make_rank(arr, A, G, sp(G), k, p, 4)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            Xr = to_rank_block(X0, ps[r])
            Gm = torch.zeros((k, k), dtype=torch.float64, device="cuda")
            ctx.gram(Xr[:ps[r].n_own], Xr[:ps[r].n_own], Gm)
            Y = torch.zeros_like(Xr)
            ritz, rank = ctx.arr_project(Xr, Y)
            res = ctx.residuals(Y, ritz[:k])
            out = (Gm.cpu().numpy(), ritz, rank, res, Y[:ps[r].n_own].cpu().numpy())
        ctx.close()
        return out

    res = run_ranks(G, work)
    for c in comms:
        c.close()
    Gref = X0.T @ X0
    for r in range(G):
        assert np.abs(res[r][0] - Gref).max() <= 1e-11 * np.abs(Gref).max()
        assert np.array_equal(res[r][1], res[0][1]), "Ritz values differ across ranks"
        assert np.array_equal(res[r][3], res[0][3]), "residuals differ across ranks"
    scale = 2 * float(np.abs(A.val).max())
    assert np.abs(res[0][1] - mu_o[:(p + 1) * k]).max() <= 1e-12 * scale * 10
    Y = np.vstack([x[4] for x in res])
    res_o = oracle.residuals(A, Y, res[0][1][:k])
    assert np.abs(res[0][3] - res_o).max() <= 1e-12 * max(1.0, res_o.max())


@pytest.mark.parametrize("kind,G", [("lap3dV", 2), ("zipf", 3), ("st27", 2), ("lap2d", 4)])
def test_dist_solve_matches_oracle(arr, kind, G):
    spec = configs.SMALL_ANALOGS[kind]
    A, spec = configs.build_config(spec)
    X0 = configs.starting_block(spec)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    planes = {"lap3dV": ("planes", spec.size, spec.size ** 2), "st27": ("planes", spec.size, spec.size ** 2),
              "lap2d": ("planes", spec.size, spec.size), "zipf": ("balanced",)}[kind]
    ps, comms, ctx_of = make_rank(arr, A, G, planes, spec.k, spec.p, spec.d, w=spec.w)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            Xr = to_rank_block(X0, ps[r])
            ev, res, info = ctx.eig_solve(Xr, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max)
            out = (ev, res, info.converged, info.outer, Xr[:ps[r].n_own, :spec.k].cpu().numpy())
        ctx.close()
        return out

    res = run_ranks(G, work)
    for c in comms:
        c.close()
    for r in range(G):
        assert res[r][2] == 1
        assert np.array_equal(res[r][0], res[0][0])
    ev = res[0][0]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) <= 1e-10
    assert res[0][1].max() <= spec.tol
    Y = np.vstack([x[4] for x in res])
    res_o = oracle.residuals(A, Y, ev)
    assert res_o.max() <= spec.tol * 1.01


def _slab_grid(kind, plan):
    """(nx, ny, nz) of a rank's z-slab for eig_set_stencil on a row partition."""
    if kind == "lap3dV":
        return 13, 13, plan.n_own // 169
    if kind == "st27":
        return 11, 11, plan.n_own // 121
    return 40, 1, plan.n_own // 40  # lap2d: x-neighbours in plane, y = the march


@pytest.mark.parametrize("kind,G", [("lap3dV", 2), ("lap3dV", 3), ("st27", 4), ("st27", 6), ("lap2d", 2),
                                    ("lap3dV", 13)])
def test_dist_stencil_path_bitwise(arr, kind, G):
    """The stencil-aware kernel on a z-slab (eig_set_stencil on a row-partitioned context:
    ghost planes below / above the owned ones, interior planes during the exchange, then the
    slab's first and last plane): bitwise the one-GPU CSR kernels' filter (same per-row FMA
    order), every rank launching the stencil kernel.  G = 6 / 13: slabs of two planes / one."""
    mk, sp = CASES[kind]
    A = mk()
    k, d = 24, 9
    X0 = synth.gaussian_block(A.n, k, 5)
    a = oracle.gershgorin_lower(A)
    b = a + 0.55 * (2 * float(np.abs(A.val).sum() / A.n * 2) - a)
    c1 = arr.eig_init(arr.to_device_csr(A), k, 1, d)
    c1.eig_set_interval(a, b)
    X1 = torch.from_numpy(X0).cuda()
    c1.filter_step(X1, normalize=False)
    ref_raw = X1.cpu().numpy()
    X1 = torch.from_numpy(X0).cuda()
    c1.filter_step(X1, normalize=True)
    ref_nrm = X1.cpu().numpy()
    c1.close()
    ps, comms, ctx_of = make_rank(arr, A, G, sp(G), k, 1, d)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            ctx.eig_set_stencil(*_slab_grid(kind, ps[r]))
            assert ctx.stencil_points > 0
            ctx.eig_set_interval(a, b)
            Xr = to_rank_block(X0, ps[r])
            ctx.filter_step(Xr, normalize=False)
            kern = ctx.last_spmm_kernel
            raw = Xr[:ps[r].n_own].cpu().numpy()
            Xr = to_rank_block(X0, ps[r], ld=k + 2)
            ctx.filter_step(Xr, normalize=True)
            nrm = Xr[:ps[r].n_own].cpu().numpy()
        ctx.close()
        return raw, nrm, kern

    res = run_ranks(G, work)
    for c in comms:
        c.close()
    assert all("stencil_kernel" in x[2] for x in res), [x[2] for x in res]
    raw = np.vstack([x[0] for x in res])
    nrm = np.vstack([x[1] for x in res])
    assert np.array_equal(raw, ref_raw), "stencil path on the z-slabs is not bitwise the one-GPU filter"
    assert np.abs(nrm - ref_nrm).max() <= 1e-14
    orc = oracle.mpm_sweep(A, a, b, d, X0)
    assert np.linalg.norm(nrm - orc) / np.linalg.norm(orc) <= 1e-12


def test_dist_stencil_rejects_non_slab(arr):
    """A traffic-balanced row block of an irregular matrix is no z-slab: EINVAL."""
    A = synth.zipf_random(5000, 3)
    ps, comms, ctx_of = make_rank(arr, A, 2, ("balanced",), 8, 1, 4)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            with pytest.raises(Exception):
                ctx.eig_set_stencil(ps[r].n_own, 1, 1)
        ctx.close()
        return True

    run_ranks(2, work)
    for c in comms:
        c.close()


@pytest.mark.parametrize("kind,G", [("lap3dV", 2), ("st27", 3)])
def test_dist_stencil_solve_matches_dense(arr, kind, G):
    """Full solve on z-slabs with the stencil path declared (filter degrees and the ARR's /
    residuals' SpMMs through the stencil kernel where it applies)."""
    spec = configs.SMALL_ANALOGS[kind]
    A, spec = configs.build_config(spec)
    X0 = configs.starting_block(spec)
    lam = np.sort(np.linalg.eigvalsh(A.to_dense()))[::-1][:spec.k]
    N = spec.size
    ps, comms, ctx_of = make_rank(arr, A, G, ("planes", N, N * N), spec.k, spec.p, spec.d, w=spec.w)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            ctx.eig_set_stencil(N, N, ps[r].n_own // (N * N))
            Xr = to_rank_block(X0, ps[r])
            ev, res, info = ctx.eig_solve(Xr, tol=spec.tol, maxit=spec.maxit, s_max=spec.s_max)
            out = (ev, res, info.converged, Xr[:ps[r].n_own, :spec.k].cpu().numpy())
        ctx.close()
        return out

    res = run_ranks(G, work)
    for c in comms:
        c.close()
    for r in range(G):
        assert res[r][2] == 1 and np.array_equal(res[r][0], res[0][0])
    ev = res[0][0]
    assert np.max(np.abs(ev - lam) / np.maximum(1, np.abs(lam))) <= 1e-10
    Y = np.vstack([x[3] for x in res])
    assert oracle.residuals(A, Y, ev).max() <= spec.tol * 1.01


def test_dist_stencil_odd_width_falls_back_to_csr(arr):
    """An odd block width is outside the stencil kernel's reach (16-byte column vectors): a
    z-slab context with the stencil declared runs the CSR tiles for that launch (exchange
    started once, ended once) and stays bitwise the one-GPU result."""
    A = synth.laplacian_3d_potential(13, 2)
    k, d, G = 23, 5, 3
    X0 = synth.gaussian_block(A.n, k, 5)
    a = oracle.gershgorin_lower(A)
    b = a + 6.0
    c1 = arr.eig_init(arr.to_device_csr(A), k, 1, d)
    c1.eig_set_interval(a, b)
    X1 = torch.from_numpy(X0).cuda()
    c1.filter_step(X1, normalize=False)
    ref = X1.cpu().numpy()
    c1.close()
    ps, comms, ctx_of = make_rank(arr, A, G, ("planes", 13, 169), k, 1, d)

    def work(r):
        ctx, s = ctx_of(r)
        with torch.cuda.stream(s):
            ctx.eig_set_stencil(13, 13, ps[r].n_own // 169)
            ctx.eig_set_interval(a, b)
            Xr = to_rank_block(X0, ps[r])
            ctx.filter_step(Xr, normalize=False)
            out = Xr[:ps[r].n_own].cpu().numpy(), ctx.last_spmm_kernel
        ctx.close()
        return out

    res = run_ranks(G, work)
    for c in comms:
        c.close()
    assert all("CSR" in x[1] for x in res), [x[1] for x in res]
    assert np.array_equal(np.vstack([x[0] for x in res]), ref)
