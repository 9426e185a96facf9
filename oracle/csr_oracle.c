/*
 * ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header or constant with paper_1507_06078_b200/csrc.
 *
 * Plain, slow, obviously-correct fp64 CPU code for the sparse part of the path
 * (arXiv 1507.06078, PAPER.md = P):
 *
 *   orc_spmm          Y = A X, plain CSR row loop summing each row in CSR order.
 *                     "AX" is the only way the method touches A (Alg. Arrabit2,
 *                     P:1527-1528 "uses A only in matrix multiplications").
 *   orc_cheb_filter   Y = T_d((A - cI)/e) X by the Chebyshev three-term
 *                     recursion rho_{d+1}(t) = 2t rho_d(t) - rho_{d-1}(t),
 *                     rho_0 = 1, rho_1 = t (Eq. cheby-poly), applied
 *                     to the mapped matrix t = (A - cI)/e with c=(a+b)/2,
 *                     e=(b-a)/2 (the affine map of Eq. rhod):
 *                       Y_0 = X
 *                       Y_1 = (A Y_0 - c Y_0) / e
 *                       Y_{j+1} = 2 (A Y_j - c Y_j) / e - Y_{j-1}
 *                     Every A*Y is a full orc_spmm into a temporary; no fusion.
 *   orc_col_norms     ||x_i||_2 of every column (MPM normalisation).
 *
 * Blocks are row-major n x w with leading dimension ld (elements).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

void orc_spmm(int64_t n, int64_t w, const int64_t *row_ptr, const int32_t *col_idx,
              const double *val, const double *X, int64_t ldx, double *Y, int64_t ldy)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double *y = Y + i * ldy;
        for (int64_t c = 0; c < w; ++c) y[c] = 0.0;
        for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
            const double a = val[p];
            const double *x = X + (int64_t)col_idx[p] * ldx;
            for (int64_t c = 0; c < w; ++c) y[c] += a * x[c];
        }
    }
}

/* Y = T_d((A - cI)/e) X.  X and Y may not alias.  Returns 0 on success. */
int orc_cheb_filter(int64_t n, int64_t w, const int64_t *row_ptr, const int32_t *col_idx,
                    const double *val, double a, double b, int32_t d,
                    const double *X, int64_t ldx, double *Y, int64_t ldy)
{
    if (!(a < b) || d < 0) return 1;
    const double c = (a + b) / 2.0;
    const double e = (b - a) / 2.0;
    const size_t sz = (size_t)n * (size_t)w;
    double *prev = (double *)malloc(sz * sizeof(double)); /* Y_{j-1} */
    double *cur = (double *)malloc(sz * sizeof(double));  /* Y_j     */
    double *ay = (double *)malloc(sz * sizeof(double));   /* A Y_j   */
    if (!prev || !cur || !ay) { free(prev); free(cur); free(ay); return 2; }
    for (int64_t i = 0; i < n; ++i)
        memcpy(cur + i * w, X + i * ldx, (size_t)w * sizeof(double));
    if (d >= 1) {
        /* Y_1 = (A Y_0 - c Y_0) / e */
        orc_spmm(n, w, row_ptr, col_idx, val, cur, w, ay, w);
        for (size_t q = 0; q < sz; ++q) {
            prev[q] = cur[q];
            cur[q] = (ay[q] - c * cur[q]) / e;
        }
    }
    for (int32_t j = 1; j < d; ++j) {
        /* Y_{j+1} = 2 (A Y_j - c Y_j) / e - Y_{j-1} */
        orc_spmm(n, w, row_ptr, col_idx, val, cur, w, ay, w);
        for (size_t q = 0; q < sz; ++q) {
            const double next = 2.0 * (ay[q] - c * cur[q]) / e - prev[q];
            prev[q] = cur[q];
            cur[q] = next;
        }
    }
    for (int64_t i = 0; i < n; ++i)
        memcpy(Y + i * ldy, cur + i * w, (size_t)w * sizeof(double));
    free(prev); free(cur); free(ay);
    return 0;
}

/* out[c] = sqrt(sum_i X[i,c]^2), summed in row order. */
void orc_col_norms(int64_t n, int64_t w, const double *X, int64_t ldx, double *out)
{
    for (int64_t c = 0; c < w; ++c) out[c] = 0.0;
    for (int64_t i = 0; i < n; ++i)
        for (int64_t c = 0; c < w; ++c) out[c] += X[i * ldx + c] * X[i * ldx + c];
    for (int64_t c = 0; c < w; ++c) out[c] = sqrt(out[c]);
}
