"""Row partition of the hot path over G GPUs (include/arrabit.h arr_dist).

North star: "A is row-partitioned with X rows co-located.  An NCCL halo
exchange (or all-gather of X for irregular sparsity) runs before each SpMM ...,
and a k x k NCCL allreduce handles the Gram blocks."  This module is host setup
only (no arithmetic of the method): it splits the rows of a global CSR into G
contiguous blocks and builds, for one rank, the local CSR with ghost columns
and the exchange plan libarrabit's eig_init_dist consumes.

Local numbering of rank r (rows [r0, r1) of A):
  - local rows 0 .. n_own-1 = global rows r0 .. r1-1, in order;
  - local columns 0 .. n_own-1 are the owned rows, n_own .. n_own+n_ghost-1 the
    ghost rows = the global columns outside [r0, r1) its rows reference, sorted
    by global id (hence grouped by owner rank, ascending);
  - each row keeps its CSR order, so every per-row sum runs in the same order
    as on one GPU (the un-normalised filter is bitwise partition independent).
Because A is structurally symmetric, the rows rank r sends to peer q (its rows
with a neighbour owned by q, ascending) are exactly q's ghost rows from r.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

TILE = 64  # rows per tile of the SpMM processing order (kTile in spmm_kernels.cu)


def bounds_balanced(row_ptr: np.ndarray, size: int, row_bytes: int = 8) -> np.ndarray:
    """Contiguous row blocks balanced by the per-degree traffic model
    12*nnz_i + row_bytes ("balanced by nnz + 8 rows")."""
    n = len(row_ptr) - 1
    cost = 12.0 * np.diff(row_ptr).astype(np.float64) + row_bytes
    cum = np.concatenate([[0.0], np.cumsum(cost)])
    targets = cum[-1] * np.arange(1, size) / size
    cuts = np.searchsorted(cum, targets, side="left")
    b = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    return np.maximum.accumulate(b)


def bounds_planes(n_planes: int, plane_rows: int, size: int) -> np.ndarray:
    """z-slabs of whole grid planes (cfg3 / cfg5: 'row-partitioned by z-slabs'),
    as even as possible: the first n_planes % size ranks get one plane more."""
    per = np.full(size, n_planes // size, dtype=np.int64)
    per[: n_planes % size] += 1
    return np.concatenate([[0], np.cumsum(per)]).astype(np.int64) * plane_rows


def _runs_to_tiles(mask: np.ndarray):
    """Contiguous runs of True in mask -> tiles of <= TILE rows (row0, len)."""
    m = np.concatenate([[False], mask, [False]]).astype(np.int8)
    d = np.diff(m)
    starts = np.flatnonzero(d == 1)
    ends = np.flatnonzero(d == -1)
    r0, ln = [], []
    for s, e in zip(starts.tolist(), ends.tolist()):
        off = np.arange(s, e, TILE, dtype=np.int64)
        r0.append(off)
        ln.append(np.minimum(TILE, e - off))
    if not r0:
        return np.zeros(0, np.int64), np.zeros(0, np.int32)
    return np.concatenate(r0).astype(np.int64), np.concatenate(ln).astype(np.int32)


@dataclass
class LocalPlan:
    rank: int
    size: int
    n_global: int
    row_begin: int
    n_own: int
    n_ghost: int
    row_ptr: np.ndarray     # int64 [n_own+1]
    col_idx: np.ndarray     # int32 [nnz_local] (local numbering)
    val: np.ndarray         # float64 [nnz_local]
    ghost_global: np.ndarray  # int64 [n_ghost] global ids of the ghost rows
    peer: np.ndarray        # int32 [npeers]
    send_off: np.ndarray    # int64 [npeers+1]
    send_rows: np.ndarray   # int32 [send_off[-1]] local owned rows, grouped by peer
    recv_off: np.ndarray    # int64 [npeers+1]
    int_row0: np.ndarray
    int_len: np.ndarray
    bnd_row0: np.ndarray
    bnd_len: np.ndarray

    @property
    def n_rows_block(self) -> int:
        """Rows of every block on this rank (owned + ghost scratch)."""
        return self.n_own + self.n_ghost

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    @property
    def n(self) -> int:  # so the plan can be handed to to_device_csr
        return self.n_own


def _yband_tiles(mask: np.ndarray, row_begin: int, nx: int, ny: int, band: int):
    """The rows of `mask` (local ids of owned rows, global id = row_begin + local) in y-band
    order on an nx x ny x nz grid (x fastest): for each band of `band` y-lines, for each
    z-plane, the band's contiguous rows of that plane, cut into tiles of <= TILE rows.  The
    same rows as _runs_to_tiles(mask), in the order that keeps a band's gathered neighbour
    rows (y +- 1 lines, z +- 1 planes) L2-resident (schedule.yband_3d)."""
    n = mask.shape[0]
    plane = nx * ny
    z0, z1 = row_begin // plane, (row_begin + n - 1) // plane + 1
    r0s, lens = [], []
    for yb in range(0, ny, band):
        h = min(band, ny - yb)
        for z in range(z0, z1):
            g0 = z * plane + yb * nx
            a, b = max(g0, row_begin), min(g0 + h * nx, row_begin + n)
            if a >= b:
                continue
            t0, tl = _runs_to_tiles(mask[a - row_begin:b - row_begin])
            r0s.append(t0 + (a - row_begin))
            lens.append(tl)
    if not r0s:
        return np.zeros(0, np.int64), np.zeros(0, np.int32)
    return np.concatenate(r0s).astype(np.int64), np.concatenate(lens).astype(np.int32)


def local_plan(A, bounds: np.ndarray, rank: int, yband: tuple | None = None) -> LocalPlan:
    """The local CSR and exchange plan of `rank` for the row blocks `bounds`
    (bounds[r] .. bounds[r+1]-1 are rank r's rows).  yband = (nx, ny, band): the interior
    tiles in y-band order of an nx x ny x nz grid (results unchanged: only the order in
    which rows are computed moves)."""
    size = len(bounds) - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    n_own = r1 - r0
    if n_own < 1:
        raise ValueError(f"rank {rank} owns no rows (bounds {bounds.tolist()}): use fewer ranks")
    p0, p1 = int(A.row_ptr[r0]), int(A.row_ptr[r1])
    rp = (A.row_ptr[r0:r1 + 1] - p0).astype(np.int64)
    cols = A.col_idx[p0:p1].astype(np.int64)
    vals = np.ascontiguousarray(A.val[p0:p1], dtype=np.float64)
    owned = (cols >= r0) & (cols < r1)
    ghost_global = np.unique(cols[~owned])
    n_ghost = int(ghost_global.shape[0])
    loc = np.empty_like(cols)
    loc[owned] = cols[owned] - r0
    loc[~owned] = n_own + np.searchsorted(ghost_global, cols[~owned])
    owner_of_ghost = np.searchsorted(bounds, ghost_global, side="right") - 1
    peers = np.unique(owner_of_ghost).astype(np.int32)
    recv_off = np.concatenate([[0], np.cumsum([np.count_nonzero(owner_of_ghost == q) for q in peers])]).astype(np.int64)
    # rows to send to q: owned rows with a column owned by q (= q's ghosts from us, A symmetric)
    row_of_entry = np.repeat(np.arange(n_own, dtype=np.int64), np.diff(rp))
    gmask = ~owned
    e_rows = row_of_entry[gmask]
    e_owner = np.searchsorted(bounds, cols[gmask], side="right") - 1
    send_lists = [np.unique(e_rows[e_owner == q]) for q in peers]
    send_off = np.concatenate([[0], np.cumsum([len(s) for s in send_lists])]).astype(np.int64)
    send_rows = (np.concatenate(send_lists) if send_lists else np.zeros(0)).astype(np.int32)
    boundary = np.zeros(n_own, dtype=bool)
    boundary[e_rows] = True
    int_row0, int_len = _runs_to_tiles(~boundary) if yband is None else _yband_tiles(~boundary, r0, *yband)
    bnd_row0, bnd_len = _runs_to_tiles(boundary)
    return LocalPlan(rank, size, int(A.n), r0, n_own, n_ghost, rp, loc.astype(np.int32), vals, ghost_global,
                     peers, send_off, send_rows, recv_off, int_row0, int_len, bnd_row0, bnd_len)


def plans(A, bounds: np.ndarray, yband: tuple | None = None) -> list[LocalPlan]:
    return [local_plan(A, bounds, r, yband) for r in range(len(bounds) - 1)]


def check_plans(ps: list[LocalPlan]) -> None:
    """Consistency of a set of plans (raises AssertionError): the rows r sends
    to q are q's ghost rows from r, in the same order; tiles cover the rows."""
    for p in ps:
        assert p.int_len.sum() + p.bnd_len.sum() == p.n_own
        cover = np.zeros(p.n_own, dtype=np.int64)
        for r0, ln in zip(np.concatenate([p.int_row0, p.bnd_row0]).tolist(),
                          np.concatenate([p.int_len, p.bnd_len]).tolist()):
            cover[r0:r0 + ln] += 1
        assert np.all(cover == 1)
        for qi, q in enumerate(p.peer.tolist()):
            pq = ps[q]
            ri = np.flatnonzero(pq.peer == p.rank)
            assert len(ri) == 1, "peer relation not symmetric"
            ri = int(ri[0])
            sent = p.send_rows[p.send_off[qi]:p.send_off[qi + 1]].astype(np.int64) + p.row_begin
            ghosts = pq.ghost_global[pq.recv_off[ri]:pq.recv_off[ri + 1]]
            assert np.array_equal(sent, ghosts), f"rank {p.rank} -> {q}: send list != ghost list"


def scatter_rows(X: np.ndarray, p: LocalPlan, ld: int | None = None) -> np.ndarray:
    """This rank's block (owned rows of the global X, then ghost rows zeroed)."""
    w = X.shape[1]
    ld = w if ld is None else ld
    out = np.zeros((p.n_rows_block, ld))
    out[:p.n_own, :w] = X[p.row_begin:p.row_begin + p.n_own]
    return out


# ---------------------------------------------------------------- column partition (Survey §8f-3)
def col_bounds(w: int, size: int) -> np.ndarray:
    """Columns [cb[r], cb[r+1]) of every n x w block on rank r: even widths (16-byte
    rows for the filter's 128-bit accesses), the remainder on the last ranks."""
    if w < 2 * size:
        raise ValueError(f"w = {w} too narrow for {size} column slices")
    per = np.full(size, (w // size) & ~1, dtype=np.int64)
    rest = w - int(per.sum())
    r = size - 1
    while rest > 0:  # hand out the remainder two columns at a time (one if w is odd)
        step = 2 if rest >= 2 else 1
        per[r] += step
        rest -= step
        r = r - 1 if r > 0 else size - 1
    return np.concatenate([[0], np.cumsum(per)]).astype(np.int64)


@dataclass
class ColSplitPlan:
    """What eig_init_colsplit needs on one rank: the row block of the internal ARR
    context (its LocalPlan, rows balanced by traffic as bounds_balanced) and the row /
    column boundaries of every rank."""
    rows: LocalPlan
    row_begins: np.ndarray  # int64 [size+1]
    col_begins: np.ndarray  # int64 [size+1]
    rank: int
    size: int

    @property
    def col_range(self):
        return int(self.col_begins[self.rank]), int(self.col_begins[self.rank + 1])


def colsplit_plan(A, w: int, size: int, rank: int, row_bounds: np.ndarray | None = None) -> ColSplitPlan:
    rb = bounds_balanced(A.row_ptr, size) if row_bounds is None else np.asarray(row_bounds, dtype=np.int64)
    return ColSplitPlan(local_plan(A, rb, rank), rb.astype(np.int64), col_bounds(w, size), rank, size)


def transpose_col2row(cols: list[np.ndarray], row_begins: np.ndarray, col_begins: np.ndarray) -> list[np.ndarray]:
    """Host reference of the all-to-all (comm.cu comm_transpose, direction 0): rank r's
    column slice (n x w_r) -> every rank's row slice (n_q x w).  Data movement only."""
    size = len(cols)
    w = int(col_begins[-1])
    out = []
    for q in range(size):
        a, b = int(row_begins[q]), int(row_begins[q + 1])
        blk = np.empty((b - a, w))
        for r in range(size):
            blk[:, col_begins[r]:col_begins[r + 1]] = cols[r][a:b]
        out.append(blk)
    return out


def transpose_row2col(rows: list[np.ndarray], row_begins: np.ndarray, col_begins: np.ndarray) -> list[np.ndarray]:
    """Inverse of transpose_col2row."""
    size = len(rows)
    n = int(row_begins[-1])
    out = []
    for r in range(size):
        c0, c1 = int(col_begins[r]), int(col_begins[r + 1])
        blk = np.empty((n, c1 - c0))
        for q in range(size):
            blk[row_begins[q]:row_begins[q + 1]] = rows[q][:, c0:c1]
        out.append(blk)
    return out
