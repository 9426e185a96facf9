"""Seeded CSR matrices and Gaussian blocks (input recipe: DESIGN.md §3).

Conventions (shared by every consumer):

* CSR with the FULL symmetric pattern stored: ``row_ptr``
  int64 ``[n+1]``, ``col_idx`` int32 ``[nnz]`` sorted ascending inside each row,
  ``val`` float64 ``[nnz]``; no duplicate entries; ``A == A^T`` bitwise.
* Grid ordering ``i = x + Nx*y + Nx*Ny*z`` (x fastest), Dirichlet truncation
  at the boundary.
* Randomness: numpy PCG64 seeded by ``SeedSequence([seed, stream, chunk])``
  over row chunks of ``ROW_CHUNK`` rows, so a block or a matrix is identical
  however it is later partitioned.  Stream 0 = the starting
  block ``X0``; stream 1 = matrix randomness.

Nothing here computes any quantity of the eigensolver.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ROW_CHUNK = 65536


@dataclass
class CSR:
    n: int
    row_ptr: np.ndarray  # int64 [n+1]
    col_idx: np.ndarray  # int32 [nnz]
    val: np.ndarray      # float64 [nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    def to_dense(self) -> np.ndarray:
        """Dense expansion (tests only, small n)."""
        a = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        a[rows, self.col_idx] = self.val
        return a

    def row_of_entry(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))


def _stencil_csr(dims, stencil, diag_extra=None, name=""):
    """CSR of a constant-coefficient stencil on an Nx*Ny*Nz grid, Dirichlet
    truncation.  ``stencil`` is a list of ((dx,dy,dz), value).  Entries of each
    row come out sorted because offsets are visited in increasing linear
    offset.  ``diag_extra`` (float64 [n]) is added to the (0,0,0) entry."""
    nx, ny, nz = dims
    n = nx * ny * nz
    idx = np.arange(n, dtype=np.int64)
    x = (idx % nx).astype(np.int32)
    y = ((idx // nx) % ny).astype(np.int32)
    z = (idx // (nx * ny)).astype(np.int32)
    offs = sorted(stencil, key=lambda t: t[0][0] + nx * t[0][1] + nx * ny * t[0][2])

    def mask_of(dx, dy, dz):
        m = np.ones(n, dtype=bool)
        if dx:
            m &= (x + dx >= 0) & (x + dx < nx)
        if dy:
            m &= (y + dy >= 0) & (y + dy < ny)
        if dz:
            m &= (z + dz >= 0) & (z + dz < nz)
        return m

    counts = np.zeros(n, dtype=np.int64)
    for (dx, dy, dz), _ in offs:
        counts += mask_of(dx, dy, dz)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    pos = row_ptr[:-1].copy()
    del counts
    for (dx, dy, dz), v in offs:
        m = mask_of(dx, dy, dz)
        rows = idx[m]
        p = pos[m]
        lin = dx + nx * dy + nx * ny * dz
        col[p] = (rows + lin).astype(np.int32)
        if (dx, dy, dz) == (0, 0, 0) and diag_extra is not None:
            val[p] = v + diag_extra[rows]
        else:
            val[p] = v
        pos[m] += 1
    return CSR(n, row_ptr, col, val, name)


def laplacian_1d(n: int) -> CSR:
    """tridiag(-1, 2, -1), Dirichlet (cfg1)."""
    return _stencil_csr((n, 1, 1), [((-1, 0, 0), -1.0), ((0, 0, 0), 2.0), ((1, 0, 0), -1.0)],
                        name=f"lap1d_{n}")


def laplacian_2d(nx: int, ny: int | None = None) -> CSR:
    """5-point Laplacian (4 on the diagonal, -1 to the 4 neighbours), Dirichlet (cfg2)."""
    ny = nx if ny is None else ny
    st = [((0, -1, 0), -1.0), ((-1, 0, 0), -1.0), ((0, 0, 0), 4.0), ((1, 0, 0), -1.0), ((0, 1, 0), -1.0)]
    return _stencil_csr((nx, ny, 1), st, name=f"lap2d_{nx}x{ny}")


def potential_uniform(n: int, seed: int) -> np.ndarray:
    """V_i ~ U[0,1) iid, chunked stream 1."""
    out = np.empty(n, dtype=np.float64)
    for c, r0 in enumerate(range(0, n, ROW_CHUNK)):
        r1 = min(n, r0 + ROW_CHUNK)
        out[r0:r1] = np.random.default_rng([seed, 1, c]).random(r1 - r0)
    return out


def laplacian_3d_potential(nx: int, seed: int | None = None) -> CSR:
    """7-point Laplacian on nx^3 (6 / -1) plus diag(V), V ~ U[0,1) (cfg3).
    ``seed=None`` gives the plain Laplacian."""
    n = nx ** 3
    st = [((0, 0, -1), -1.0), ((0, -1, 0), -1.0), ((-1, 0, 0), -1.0), ((0, 0, 0), 6.0),
          ((1, 0, 0), -1.0), ((0, 1, 0), -1.0), ((0, 0, 1), -1.0)]
    v = None if seed is None else potential_uniform(n, seed)
    return _stencil_csr((nx, nx, nx), st, diag_extra=v,
                        name=f"lap3d_{nx}" + ("" if seed is None else f"_V{seed}"))


def stencil27_3d(nx: int) -> CSR:
    """27-point stencil on nx^3: centre 26, the 26 neighbours -1, Dirichlet (cfg5)."""
    st = []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                st.append(((dx, dy, dz), 26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0))
    return _stencil_csr((nx, nx, nx), st, name=f"st27_{nx}")


def diagonal(d: np.ndarray) -> CSR:
    n = len(d)
    return CSR(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
               np.asarray(d, dtype=np.float64).copy(), name=f"diag_{n}")


def from_dense(a: np.ndarray, name: str = "dense") -> CSR:
    """CSR of the non-zeros of a dense symmetric matrix (tests)."""
    n = a.shape[0]
    rows, cols = np.nonzero(a)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return CSR(n, row_ptr, cols.astype(np.int32), a[rows, cols].astype(np.float64), name)


def zipf_random(n: int, seed: int, dmin: int = 2, dmax: int = 256, expo: float = 2.0) -> CSR:
    """Random sparse symmetric matrix of cfg4.

    Per row i: degree d_i ~ Zipf law truncated to {dmin..dmax}, P(d) ∝ d^-expo;
    d_i partners j != i uniform with replacement, values N(0,1) -> B (duplicate
    (i,j) summed).  S = B + B^T (each off-diagonal S_ij is a sum of exactly two
    B terms, so S is bitwise symmetric); A_ii = sum_j |S_ij| (SPD by Gershgorin).
    """
    support = np.arange(dmin, dmax + 1)
    prob = support.astype(np.float64) ** (-expo)
    prob /= prob.sum()
    rows_l, cols_l, vals_l = [], [], []
    for c, r0 in enumerate(range(0, n, ROW_CHUNK)):
        r1 = min(n, r0 + ROW_CHUNK)
        rng = np.random.default_rng([seed, 1, c])
        deg = rng.choice(support, size=r1 - r0, p=prob)
        tot = int(deg.sum())
        r = np.repeat(np.arange(r0, r1, dtype=np.int64), deg)
        j = rng.integers(0, n - 1, size=tot, dtype=np.int64)
        j += (j >= r)
        v = rng.standard_normal(tot)
        rows_l.append(r); cols_l.append(j); vals_l.append(v)
    r = np.concatenate(rows_l); j = np.concatenate(cols_l); v = np.concatenate(vals_l)
    del rows_l, cols_l, vals_l
    # dedup B
    key = r * n + j
    del r, j
    ukey, inv = np.unique(key, return_inverse=True)
    bv = np.bincount(inv, weights=v)
    del key, inv, v
    bi = ukey // n
    bj = ukey % n
    del ukey
    # S = B + B^T
    key = np.concatenate([bi * n + bj, bj * n + bi])
    sv = np.concatenate([bv, bv])
    del bi, bj, bv
    order = np.argsort(key, kind="stable")
    key = key[order]
    sv = sv[order]
    del order
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.nonzero(first)[0]
    skey = key[starts]
    sval = np.add.reduceat(sv, starts)  # at most 2 terms per key: commutative -> symmetric
    del key, sv, first, starts
    si = skey // n
    sj = (skey % n).astype(np.int32)
    del skey
    # diagonal = row abs-sum, inserted in sorted position
    absv = np.abs(sval)
    cnt = np.bincount(si, minlength=n)
    off_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=off_ptr[1:])
    diag = np.zeros(n)
    nz = cnt > 0
    diag[nz] = np.add.reduceat(absv, off_ptr[:-1][nz])
    del absv
    row_ptr = off_ptr + np.arange(n + 1, dtype=np.int64)
    nnz = int(row_ptr[-1])
    col = np.empty(nnz, dtype=np.int32)
    val = np.empty(nnz, dtype=np.float64)
    # number of off-diagonal entries of row i with column < i
    lt = (sj.astype(np.int64) < si)
    nlt = np.bincount(si[lt], minlength=n)
    # destination of each off-diagonal entry: row_ptr[i] + rank_in_row + (1 if col > i)
    rank_in_row = np.arange(len(si), dtype=np.int64) - off_ptr[si]
    dest = row_ptr[si] + rank_in_row + (~lt)
    col[dest] = sj
    val[dest] = sval
    dpos = row_ptr[:-1] + nlt
    col[dpos] = np.arange(n, dtype=np.int32)
    val[dpos] = diag
    return CSR(n, row_ptr, col, val, name=f"zipf_{n}_s{seed}")


def gaussian_block_rows(n: int, w: int, seed: int, r0: int, r1: int, stream: int = 0) -> np.ndarray:
    """Rows [r0, r1) of the n x w iid N(0,1) block of ``seed`` (stream 0; guard
    columns use stream 2).
    Chunk c covers rows [c*ROW_CHUNK, (c+1)*ROW_CHUNK) and is drawn from
    default_rng([seed, 0, c]).standard_normal((rows, w))."""
    out = np.empty((r1 - r0, w), dtype=np.float64)
    c0 = r0 // ROW_CHUNK
    c1 = (r1 - 1) // ROW_CHUNK if r1 > r0 else c0 - 1
    for c in range(c0, c1 + 1):
        a = c * ROW_CHUNK
        b = min(n, a + ROW_CHUNK)
        blk = np.random.default_rng([seed, stream, c]).standard_normal((b - a, w))
        lo, hi = max(a, r0), min(b, r1)
        out[lo - r0:hi - r0] = blk[lo - a:hi - a]
    return out


def gaussian_block(n: int, w: int, seed: int, stream: int = 0) -> np.ndarray:
    """The full n x w Gaussian block (row-major, C-contiguous)."""
    return gaussian_block_rows(n, w, seed, 0, n, stream)
