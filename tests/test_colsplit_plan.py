"""Host logic of the column-partitioned mode (eig_init_colsplit, Survey §8f-3) on CPU:
the column / row boundaries, the reference transposes, and the whole protocol under
torch.distributed gloo with world size 2 - a column-local MPM sweep (no exchange: MPM
filters every column independently), the col->row all-to-all by point-to-point
messages, the ARR Gram as a row-sum allreduce, and the row->col transpose back - against
the oracle's single-process sweep and Gram."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from paper_1507_06078_b200 import partition as pt


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("w,size", [(22, 2), (36, 3), (37, 4), (1100, 8), (282, 8), (9, 4)])
def test_col_bounds(w, size):
    cb = pt.col_bounds(w, size)
    assert cb[0] == 0 and cb[-1] == w and len(cb) == size + 1
    widths = np.diff(cb)
    assert np.all(widths >= 2) and widths.max() - widths.min() <= 2
    assert np.sum(widths % 2 == 1) <= 1  # at most one odd slice (odd w)


def test_transposes_round_trip():
    rng = np.random.default_rng(0)
    n, w, size = 57, 13, 3
    X = rng.standard_normal((n, w))
    rb = np.array([0, 20, 31, 57])
    cb = pt.col_bounds(w, size)
    cols = [X[:, cb[r]:cb[r + 1]].copy() for r in range(size)]
    rows = pt.transpose_col2row(cols, rb, cb)
    for q in range(size):
        assert np.array_equal(rows[q], X[rb[q]:rb[q + 1]])
    back = pt.transpose_row2col(rows, rb, cb)
    for r in range(size):
        assert np.array_equal(back[r], cols[r])


def _col2row(dist, cols_local, rb, cb, rank, size):
    """col -> row transpose with point-to-point messages (the NCCL send/recv pattern)."""
    import torch
    w = int(cb[-1])
    nr = int(rb[rank + 1] - rb[rank])
    out = np.empty((nr, w))
    reqs, bufs = [], []
    for q in range(size):
        piece = torch.from_numpy(np.ascontiguousarray(cols_local[rb[q]:rb[q + 1]]))
        if q == rank:
            out[:, cb[rank]:cb[rank + 1]] = piece.numpy()
            continue
        rbuf = torch.empty((nr, int(cb[q + 1] - cb[q])), dtype=torch.float64)
        bufs.append((q, rbuf, piece))
        reqs.append(dist.isend(piece, q))
        reqs.append(dist.irecv(rbuf, q))
    for r in reqs:
        r.wait()
    for q, rbuf, _ in bufs:
        out[:, cb[q]:cb[q + 1]] = rbuf.numpy()
    return out


def _worker(rank, size, port, out_q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        A = synth.zipf_random(3000, 3)
        w, d = 10, 6
        plan = pt.colsplit_plan(A, w, size, rank)
        c0, c1 = plan.col_range
        X0 = synth.gaussian_block(A.n, w, 4)
        a = oracle.gershgorin_lower(A)
        b = a + 0.6 * (4.0 * float(np.abs(A.val).max()) - a)
        Xc = oracle.mpm_sweep(A, a, b, d, X0[:, c0:c1])  # column-local: no communication
        Xr = _col2row(dist, Xc, plan.row_begins, plan.col_begins, rank, size)
        assert Xr.shape == (plan.rows.n_own, w)
        G = torch.from_numpy(Xr.T @ Xr)
        dist.all_reduce(G)  # the ARR Gram over the row blocks
        gathered = [None] * size if rank == 0 else None
        dist.gather_object((plan.rows.row_begin, Xr), gathered, dst=0)
        if rank == 0:
            ref = oracle.mpm_sweep(A, a, b, d, X0)
            Xg = np.zeros_like(ref)
            for r0, blk in gathered:
                Xg[r0:r0 + blk.shape[0]] = blk
            out_q.put((float(np.abs(Xg - ref).max()), float(np.abs(G.numpy() - ref.T @ ref).max())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_colsplit_protocol():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    xerr, gerr = q.get(timeout=5)
    assert xerr == 0.0  # the column-local sweep is bitwise the full sweep's columns
    assert gerr <= 1e-12
