"""Input generators: CSR invariants and closed-form sizes (SURVEY.md §8c-5 'Generators')."""
import numpy as np
import pytest

import synth
from synth import configs


def _check_csr(A):
    n = A.n
    assert A.row_ptr.dtype == np.int64 and A.col_idx.dtype == np.int32 and A.val.dtype == np.float64
    assert A.row_ptr[0] == 0 and len(A.row_ptr) == n + 1
    assert np.all(np.diff(A.row_ptr) >= 0)
    rows = A.row_of_entry()
    # sorted strictly inside each row (no duplicates), in range
    same = np.diff(rows) == 0
    assert np.all(np.diff(A.col_idx.astype(np.int64))[same] > 0)
    assert A.col_idx.min() >= 0 and A.col_idx.max() < n
    # bitwise symmetric
    key = rows * n + A.col_idx
    keyT = A.col_idx.astype(np.int64) * n + rows
    o = np.argsort(keyT)
    assert np.array_equal(key, keyT[o])
    assert np.array_equal(A.val, A.val[o])


@pytest.mark.parametrize("build,nnz", [
    (lambda: synth.laplacian_1d(2000), 3 * 2000 - 2),                       # cfg1: 5,998
    (lambda: synth.laplacian_2d(300), 5 * 90000 - 4 * 300),                 # cfg2: 448,800
    (lambda: synth.laplacian_3d_potential(30, 2), 7 * 30 ** 3 - 6 * 30 ** 2),
    (lambda: synth.stencil27_3d(12), (3 * 12 - 2) ** 3),
])
def test_stencil_nnz_closed_form(build, nnz):
    A = build()
    _check_csr(A)
    assert A.nnz == nnz


def test_cfg3_nnz_closed_form():
    A = synth.laplacian_3d_potential(100, 2)
    assert A.nnz == 6_940_000


def test_laplacian_row_sums_and_potential():
    A = synth.laplacian_2d(20)
    s = np.bincount(A.row_of_entry(), weights=A.val, minlength=A.n).reshape(20, 20)
    assert np.all(s[1:-1, 1:-1] == 0)
    B = synth.laplacian_3d_potential(10, 2)
    L = synth.laplacian_3d_potential(10, None)
    V = synth.generators.potential_uniform(1000, 2)
    assert np.all((V >= 0) & (V < 1))
    assert np.array_equal(B.col_idx, L.col_idx)
    d = B.to_dense() - L.to_dense()
    assert np.allclose(d, np.diag(V), atol=0, rtol=0) or np.max(np.abs(d - np.diag(V))) < 1e-15
    C = synth.stencil27_3d(6)
    s = np.bincount(C.row_of_entry(), weights=C.val, minlength=C.n).reshape(6, 6, 6)
    assert np.all(s[1:-1, 1:-1, 1:-1] == 0)


def test_zipf_generator():
    A = synth.zipf_random(20000, 3)
    _check_csr(A)
    rows = A.row_of_entry()
    isd = A.col_idx == rows
    assert isd.sum() == A.n
    off = np.bincount(rows[~isd], weights=np.abs(A.val[~isd]), minlength=A.n)
    diag = np.zeros(A.n)
    diag[rows[isd]] = A.val[isd]
    assert np.allclose(diag, off, rtol=1e-13, atol=0)  # same terms, summation order differs
    per_row = A.nnz / A.n
    assert 15.5 < per_row < 18.5, per_row  # "mean ≈16" + diagonal
    assert np.diff(A.row_ptr).max() <= 2 * 256 + 1


def test_gaussian_block_is_chunk_invariant():
    n, w = 70000, 3
    full = synth.gaussian_block(n, w, 7)
    part = synth.gaussian_block_rows(n, w, 7, 65000, 66000)
    assert np.array_equal(full[65000:66000], part)
    assert full.flags.c_contiguous and full.shape == (n, w)
    assert abs(full.mean()) < 0.02 and abs(full.std() - 1) < 0.02


def test_config_table():
    assert [configs.CONFIGS[i].n for i in range(1, 6)] == [2000, 90000, 10 ** 6, 4 * 10 ** 6, 256 ** 3]
    assert [configs.CONFIGS[i].k for i in range(1, 6)] == [20, 200, 500, 1000, 256]
    assert [configs.CONFIGS[i].d for i in range(1, 6)] == [10, 20, 20, 15, 30]
    assert [configs.CONFIGS[i].p for i in range(1, 6)] == [1, 1, 2, 1, 2]
    assert [configs.CONFIGS[i].seed for i in range(1, 6)] == [0, 1, 2, 3, 4]
