"""cuBLAS (DGEMM via torch, DSYRK via ctypes) against libarrabit's DMMA Gram / GEMM on the
ARR shapes of the cfg2 / cfg3 solves.  Shapes: the Gram X^T Y of the
orthonormalisation and CGS passes (m1 x m2 = jw x w), the symmetric X^T X, and the
update / Ritz GEMM X B (n x m1 by m1 x m2).

    python scripts/micro_gram_shapes.py [--no-cublas | --cublas-only]   (ARRABIT_DMMA_TILE=v: tile variant v)
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_06078_b200 as arr  # noqa: E402

SHAPES = [(90000, 220, 220), (90000, 440, 220), (1000000, 550, 550), (1000000, 1100, 550), (1000000, 1650, 550)]


def t(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cublas_syrk():
    """C (w x w, col-major upper) = X^T X for row-major X (n x w) = A A^T with A = X viewed
    column-major w x n."""
    lib = None
    for name in ("libcublas.so.12", "libcublas.so"):
        try:
            lib = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if lib is None:
        return None
    h = ctypes.c_void_p()
    if lib.cublasCreate_v2(ctypes.byref(h)) != 0:
        return None
    one, zero = ctypes.c_double(1.0), ctypes.c_double(0.0)

    def syrk(X, C):
        n, w = X.shape
        lib.cublasSetStream_v2(h, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        # uplo = CUBLAS_FILL_MODE_UPPER (1), trans = CUBLAS_OP_N (0)
        st = lib.cublasDsyrk_v2(h, 1, 0, w, n, ctypes.byref(one), ctypes.c_void_p(X.data_ptr()), w,
                                ctypes.byref(zero), ctypes.c_void_p(C.data_ptr()), w)
        assert st == 0, st
    return syrk


class Diag:  # identity CSR of order n: the context only needs A.n for the dense products
    def __init__(self, n):
        self.n = n
        self.row_ptr = np.arange(n + 1)
        self.col_idx = np.arange(n)
        self.val = np.ones(n)


def main():
    cub = "--no-cublas" not in sys.argv
    tag = f"arr(gemm variant {os.environ.get('ARRABIT_DMMA_TILE', '0')}, gram variant {os.environ.get('ARRABIT_DMMA_GRAM', os.environ.get('ARRABIT_DMMA_TILE', '7'))})"
    only_cublas = "--cublas-only" in sys.argv
    syrk = cublas_syrk() if cub else None
    for n, m1, m2 in SHAPES:
        X = torch.randn(n, m1, dtype=torch.float64, device="cuda")
        Y = torch.randn(n, m2, dtype=torch.float64, device="cuda")
        B = torch.randn(m1, m2, dtype=torch.float64, device="cuda")
        O = torch.empty(n, m2, dtype=torch.float64, device="cuda")
        fl = 2.0 * n * m1 * m2
        if cub:
            ms = t(lambda: X.T @ Y)
            print(f"cuBLAS DGEMM X^T Y  n={n} {m1}x{m2}: {ms*1e3:8.0f} us {fl/ms/1e9:5.1f} TF/s", flush=True)
            ms = t(lambda: X @ B)
            print(f"cuBLAS DGEMM X B    n={n} {m1}->{m2}: {ms*1e3:8.0f} us {fl/ms/1e9:5.1f} TF/s", flush=True)
            if syrk and m1 == m2:
                C = torch.empty(m1, m1, dtype=torch.float64, device="cuda")
                ms = t(lambda: syrk(X, C))
                print(f"cuBLAS DSYRK X^T X  n={n} {m1}: {ms*1e3:8.0f} us {fl/2/ms/1e9:5.1f} TF/s (n w(w+1) flops)"
                      f"  {fl/ms/1e9:5.1f} TF/s (2nw^2)", flush=True)
        if only_cublas:
            continue
        w = max(m1, m2)
        ctx = arr.eig_init(arr.to_device_csr(Diag(n)), w, 2, 2, w=w)
        G = torch.empty(m1, m2, dtype=torch.float64, device="cuda")
        ms = t(lambda: ctx.gram(X, Y, G))
        ref = X.T @ Y
        err = float((G - ref).abs().max() / ref.abs().max())
        print(f"{tag} gram X^T Y    n={n} {m1}x{m2}: {ms*1e3:8.0f} us {fl/ms/1e9:5.1f} TF/s  (max rel dev from cuBLAS {err:.1e})", flush=True)
        if m1 == m2:
            ms = t(lambda: ctx.gram(X, X, G))
            print(f"{tag} gram X^T X    n={n} {m1}: {ms*1e3:8.0f} us {fl/2/ms/1e9:5.1f} TF/s (n w(w+1) flops)"
                  f"  {fl/ms/1e9:5.1f} TF/s (2nw^2)", flush=True)
        ms = t(lambda: ctx.gemm(X, B, O))
        ref = X @ B
        err = float((O - ref).abs().max() / ref.abs().max())
        print(f"{tag} gemm X B      n={n} {m1}->{m2}: {ms*1e3:8.0f} us {fl/ms/1e9:5.1f} TF/s  (max rel dev from cuBLAS {err:.1e})", flush=True)
        ctx.close()
        del X, Y, B, O, G
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
