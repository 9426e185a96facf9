"""Row-tile processing orders for libarrabit's SpMM (eig_set_schedule).

For a d-dimensional stencil on an Nx x Ny x Nz grid stored x-fastest, natural
order gathers row i's +z neighbour ~Nx*Ny rows before it is reused by its -z
neighbour, a reuse distance of 2*Nx*Ny rows of Y_j (80 MB for cfg3, 256 MB for
cfg5 per degree) that exceeds L2.  Sweeping y-bands of `by` grid lines, z-major
inside each band, shrinks it to 2*by*Nx rows (SURVEY.md §7 hard part 1(a)).
Only the processing order changes; every row's arithmetic is identical.
"""
from __future__ import annotations

import numpy as np

TILE = 64  # rows per tile (kTile in spmm_kernels.cu)


def natural(n: int):
    r0 = np.arange(0, n, TILE, dtype=np.int64)
    return r0, np.minimum(TILE, n - r0).astype(np.int32)


def ranges_to_tiles(starts: np.ndarray, lens: np.ndarray, tile: int = TILE):
    """Split contiguous row ranges (in processing order) into tiles of <= tile rows."""
    r0_list, len_list = [], []
    for s, l in zip(starts.tolist(), lens.tolist()):
        off = np.arange(0, l, tile, dtype=np.int64)
        r0_list.append(s + off)
        len_list.append(np.minimum(tile, l - off))
    return np.concatenate(r0_list).astype(np.int64), np.concatenate(len_list).astype(np.int32)


def yband_3d(nx: int, ny: int, nz: int, by: int, tile: int = TILE):
    """for each y-band of `by` lines: for z: the contiguous rows of that band at z."""
    starts, lens = [], []
    for yb in range(0, ny, by):
        h = min(by, ny - yb)
        for z in range(nz):
            starts.append(nx * yb + nx * ny * z)
            lens.append(nx * h)
    return ranges_to_tiles(np.array(starts, dtype=np.int64), np.array(lens, dtype=np.int64), tile)


def auto_band(nx: int, ny: int, w: int, l2_bytes: float = 126e6, frac: float = 0.25) -> int:
    """Largest band height whose reuse window (2*by*nx rows of 8w bytes) uses at
    most `frac` of L2 (the rest holds the Y_{j-1}/Y_{j+1} streams and CSR)."""
    by = int(frac * l2_bytes / (2 * nx * 8 * w))
    return max(1, min(ny, by))
