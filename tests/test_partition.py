"""Host logic of the multi-GPU path (include/arrabit.h arr_dist):
the row partition and exchange plan of paper_1507_06078_b200/partition.py,
checked on CPU.  The world-size-2 gloo test runs the exchange protocol the
library implements (send the planned rows, receive into the ghost rows, sum the
Gram / column-norm partials over ranks) between two processes and checks a
distributed MPM sweep and Gram against the oracle's global ones."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synth
from paper_1507_06078_b200 import partition as pt

SMALL = {
    "lap1d": (lambda: synth.laplacian_1d(300), None),
    "lap2d": (lambda: synth.laplacian_2d(24), (24, 24)),
    "lap3dV": (lambda: synth.laplacian_3d_potential(9, 2), (9, 81)),
    "zipf": (lambda: synth.zipf_random(1500, 3), None),
    "st27": (lambda: synth.stencil27_3d(8), (8, 64)),
}


def _bounds(A, planes, G):
    if planes is None:
        return pt.bounds_balanced(A.row_ptr, G)
    return pt.bounds_planes(planes[0], planes[1], G)


def _local_matrix(p):
    return sp.csr_matrix((p.val, p.col_idx, p.row_ptr), shape=(p.n_own, p.n_own + p.n_ghost))


@pytest.mark.parametrize("kind", list(SMALL))
@pytest.mark.parametrize("G", [1, 2, 3, 5])
def test_plan_consistent_and_local_spmm_exact(kind, G):
    mk, planes = SMALL[kind]
    A = mk()
    ps = pt.plans(A, _bounds(A, planes, G))
    pt.check_plans(ps)
    assert sum(p.n_own for p in ps) == A.n
    rng = np.random.default_rng(7)
    X = rng.standard_normal((A.n, 5))
    Y = oracle.spmm(A, X)
    for p in ps:
        # the local block: owned rows then the ghost rows (what the exchange delivers)
        Xl = np.vstack([X[p.row_begin:p.row_begin + p.n_own], X[p.ghost_global]])
        Yl = _local_matrix(p) @ Xl
        np.testing.assert_allclose(Yl, Y[p.row_begin:p.row_begin + p.n_own], rtol=0, atol=1e-13)
        # CSR order of every row is preserved (per-row sums in the same order as on one GPU)
        gcols = p.col_idx.astype(np.int64) + p.row_begin
        gh = p.col_idx >= p.n_own
        gcols[gh] = p.ghost_global[p.col_idx[gh] - p.n_own]
        np.testing.assert_array_equal(gcols, A.col_idx[A.row_ptr[p.row_begin]:A.row_ptr[p.row_begin + p.n_own]])


def test_boundary_rows_are_exactly_those_with_ghost_columns():
    A = synth.laplacian_3d_potential(9, 2)
    ps = pt.plans(A, pt.bounds_planes(9, 81, 3))
    mid = ps[1]
    # z-slab of 3 planes: the first and last plane reference the neighbours' planes
    bnd = np.zeros(mid.n_own, bool)
    for r0, ln in zip(mid.bnd_row0, mid.bnd_len):
        bnd[r0:r0 + ln] = True
    expect = np.zeros(mid.n_own, bool)
    expect[:81] = True
    expect[-81:] = True
    np.testing.assert_array_equal(bnd, expect)
    # halo = one plane from each neighbour, contiguous send ranges
    assert mid.n_ghost == 162 and list(mid.peer) == [0, 2]
    np.testing.assert_array_equal(mid.send_rows[:81], np.arange(81))
    np.testing.assert_array_equal(mid.send_rows[81:], np.arange(mid.n_own - 81, mid.n_own))


def test_bounds():
    np.testing.assert_array_equal(pt.bounds_planes(100, 10, 8) // 10, [0, 13, 26, 39, 52, 64, 76, 88, 100])
    rp = np.arange(0, 101, dtype=np.int64)  # 100 rows of 1 nnz
    b = pt.bounds_balanced(rp, 4)
    np.testing.assert_array_equal(b, [0, 25, 50, 75, 100])
    with pytest.raises(ValueError):
        pt.plans(synth.laplacian_1d(10), pt.bounds_planes(2, 5, 3))  # an empty rank


# ---------------------------------------------------------------- gloo, world size 2
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(dist, p, Y):
    """Fill the ghost rows of Y (n_own+n_ghost rows): send the planned rows to
    each peer, receive each peer's rows into Y[n_own + recv_off[q] : ...]."""
    import torch
    reqs = []
    bufs = []
    for qi, q in enumerate(p.peer.tolist()):
        rows = p.send_rows[p.send_off[qi]:p.send_off[qi + 1]]
        sb = torch.from_numpy(np.ascontiguousarray(Y[rows]))
        rb = torch.empty((int(p.recv_off[qi + 1] - p.recv_off[qi]), Y.shape[1]), dtype=torch.float64)
        bufs.append((qi, rb, sb))
        reqs.append(dist.isend(sb, q))
        reqs.append(dist.irecv(rb, q))
    for r in reqs:
        r.wait()
    for qi, rb, _ in bufs:
        Y[p.n_own + p.recv_off[qi]:p.n_own + p.recv_off[qi + 1]] = rb.numpy()


def _worker(rank, size, port, kind, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        mk, planes = SMALL[kind]
        A = mk()
        p = pt.local_plan(A, _bounds(A, planes, size), rank)
        Al = _local_matrix(p)
        w, d = 6, 7
        X0 = synth.gaussian_block(A.n, w, 11)
        a = oracle.gershgorin_lower(A)
        b = a + 0.6 * (4.0 * float(np.abs(A.val).max()) - a)
        c, e = (a + b) / 2, (b - a) / 2
        # distributed MPM sweep (one filter application + column normalisation)
        Yprev = None
        Y = pt.scatter_rows(X0, p)
        for j in range(d):
            _exchange(dist, p, Y)
            AY = Al @ Y
            nxt = np.zeros_like(Y)
            if j == 0:
                nxt[:p.n_own] = (AY - c * Y[:p.n_own]) / e
            else:
                nxt[:p.n_own] = (2 / e) * (AY - c * Y[:p.n_own]) - Yprev[:p.n_own]
            Yprev, Y = Y, nxt
        ss = torch.from_numpy((Y[:p.n_own] ** 2).sum(axis=0))
        dist.all_reduce(ss)  # column sums of squares over ranks
        Yn = Y[:p.n_own] / np.sqrt(ss.numpy())
        G = torch.from_numpy(Yn.T @ Yn)
        dist.all_reduce(G)  # the Gram allreduce
        gathered = [None] * size if rank == 0 else None
        dist.gather_object((p.row_begin, Yn), gathered, dst=0)
        if rank == 0:
            ref = oracle.mpm_sweep(A, a, b, d, X0)
            Yg = np.zeros_like(ref)
            for r0, blk in gathered:
                Yg[r0:r0 + blk.shape[0]] = blk
            err = np.linalg.norm(Yg - ref) / np.linalg.norm(ref)
            gerr = np.abs(G.numpy() - ref.T @ ref).max()
            out_q.put((err, gerr))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["lap2d", "zipf", "st27"])
def test_gloo_world2_distributed_sweep_matches_oracle(kind):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    err, gerr = q.get(timeout=5)
    assert err <= 1e-12, err
    assert gerr <= 1e-12, gerr


@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("band", [1, 3, 9])
def test_yband_interior_order_same_rows(G, band):
    """z-slab plans with the interior tiles in y-band order (bench.py's N > 1 default on the
    3-D grids): the same interior rows, each exactly once, tiles <= TILE rows, and the order
    is band-major (all planes of a band before the next band)."""
    N = 9
    A = synth.laplacian_3d_potential(N, 2)
    bounds = pt.bounds_planes(N, N * N, G)
    nat = pt.plans(A, bounds)
    yb = pt.plans(A, bounds, yband=(N, N, band))
    pt.check_plans(yb)
    for p, q in zip(nat, yb):
        assert np.array_equal(p.bnd_row0, q.bnd_row0) and np.array_equal(p.bnd_len, q.bnd_len)
        rows_p = np.concatenate([np.arange(r, r + ln) for r, ln in zip(p.int_row0, p.int_len)] or [np.zeros(0, int)])
        rows_q = np.concatenate([np.arange(r, r + ln) for r, ln in zip(q.int_row0, q.int_len)] or [np.zeros(0, int)])
        assert len(rows_q) == len(set(rows_q.tolist())) and np.array_equal(np.sort(rows_p), np.sort(rows_q))
        assert (q.int_len <= pt.TILE).all()
        if len(rows_q):
            yline = ((rows_q + q.row_begin) // N) % N
            assert (np.diff(yline // band) >= 0).all(), "band-major order"


@pytest.mark.parametrize("kind,yband", [("lap2d", None), ("lap3dV", None), ("st27", None), ("lap3dV", (9, 9, 3))])
@pytest.mark.parametrize("G", [2, 3, 4])
def test_zslab_plans_have_whole_ghost_planes_lower_first(kind, yband, G):
    """What eig_set_stencil on a row-partitioned context relies on (include/arrabit.h): on
    a bounds_planes partition of a stencil operator every rank owns whole planes, its ghost
    rows are exactly the plane below (from lower ranks, first in the block) and / or the
    plane above, and the plan's boundary tiles are exactly the slab's first / last plane
    (the rows the stencil path hands to the CSR kernels after the exchange)."""
    mk, planes = SMALL[kind]
    A = mk()
    nplanes, nxy = planes
    ps = pt.plans(A, pt.bounds_planes(nplanes, nxy, G), yband=yband)
    for p in ps:
        assert p.n_own % nxy == 0 and p.n_own >= nxy
        lo = p.rank > 0
        hi = p.rank < G - 1
        want = []
        if lo:
            want.append(np.arange(p.row_begin - nxy, p.row_begin))
        if hi:
            want.append(np.arange(p.row_begin + p.n_own, p.row_begin + p.n_own + nxy))
        np.testing.assert_array_equal(p.ghost_global, np.concatenate(want) if want else np.empty(0, dtype=np.int64))
        # peers in rank order: the lower neighbour's rows are received first
        cnt = np.diff(p.recv_off)
        assert [int(q) for q in p.peer] == sorted(int(q) for q in p.peer)
        assert int(cnt[p.peer < p.rank].sum()) == (nxy if lo else 0)
        assert int(cnt[p.peer > p.rank].sum()) == (nxy if hi else 0)
        bnd = np.zeros(p.n_own, dtype=bool)
        for r0, ln in zip(p.bnd_row0, p.bnd_len):
            assert not bnd[r0:r0 + ln].any()
            bnd[r0:r0 + ln] = True
        ends = np.zeros(p.n_own, dtype=bool)
        if lo:
            ends[:nxy] = True
        if hi:
            ends[p.n_own - nxy:] = True
        np.testing.assert_array_equal(bnd, ends)
