// Tall-skinny fp64 contractions of the ARR step (Alg. RR, Alg. ARR
// P:537-540) on the FP64 tensor cores of sm_100a: mma.sync.m8n8k4.f64 (DMMA;
// tcgen05 has no f64 kind).  Gram products are split over rows with a fixed-
// order reduction of the partial tiles (deterministic, no atomics).
#include <math.h>
#include <stdlib.h>

#include <cmath>

#include "internal.cuh"

#ifndef ARR_DMMA_CA
#define ARR_DMMA_CA 1  // cp.async multi-stage pipelines for the Gram / GEMM kernels
#endif

namespace {

constexpr int TILE = 64;   // CTA tile edge (4 warps, 2x2, 32x32 each)
constexpr int KS = 16;     // rows (Gram) / k-columns (GEMM) per stage
constexpr int PAD = 4;     // smem padding (doubles): conflict-free fragment loads
constexpr int THREADS = 128;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// partials[split][a][b] (ld = m2) = sum_{i in slab} X[i, a] * Y[i, b]
__global__ void __launch_bounds__(THREADS) gram_kernel(const double *__restrict__ X, int64_t ldx, int m1,
                                                       const double *__restrict__ Y, int64_t ldy, int m2,
                                                       int64_t n, int64_t rows_per_split, bool sym,
                                                       double *__restrict__ part) {
    const int ta = blockIdx.x, tb = blockIdx.y, split = blockIdx.z;
    if (sym && tb < ta) return;
    const int a0 = ta * TILE, b0 = tb * TILE;
    const int64_t k0 = (int64_t)split * rows_per_split;
    int64_t k1 = k0 + rows_per_split;
    if (k1 > n) k1 = n;
    __shared__ double Xs[2][KS][TILE + PAD];
    __shared__ double Ys[2][KS][TILE + PAD];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    constexpr int PER = KS * TILE / THREADS;  // 8 elements per operand per thread
    double rx[PER], ry[PER];
    auto gload = [&](int64_t kb) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + q * THREADS;
            const int rr = idx / TILE, cc = idx % TILE;
            const int64_t row = kb + rr;
            const bool rok = row < k1;
            rx[q] = (rok && a0 + cc < m1) ? __ldg(X + row * ldx + a0 + cc) : 0.0;
            ry[q] = (rok && b0 + cc < m2) ? __ldg(Y + row * ldy + b0 + cc) : 0.0;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + q * THREADS;
            const int rr = idx / TILE, cc = idx % TILE;
            Xs[buf][rr][cc] = rx[q];
            Ys[buf][rr][cc] = ry[q];
        }
    };
    // warps whose 32 x 32 sub-tile is out of range, or (symmetric) strictly below
    // the diagonal, only help with the loads (their results are never read)
    const bool work = (a0 + wm * 32 < m1) && (b0 + wn * 32 < m2) && !(sym && ta == tb && wm > wn);
    if (k0 < k1) {
        gload(k0);
        sstore(0);
        __syncthreads();
        int buf = 0;
        for (int64_t kb = k0; kb < k1; kb += KS) {
            const bool more = kb + KS < k1;
            if (more) gload(kb + KS);
#pragma unroll
            for (int kk = 0; kk < KS / 4; ++kk) {
                if (!work) continue;
                double af[4], bf[4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = Xs[buf][kk * 4 + (lane & 3)][wm * 32 + mt * 8 + (lane >> 2)];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) bf[nt] = Ys[buf][kk * 4 + (lane & 3)][wn * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
            }
            if (more) {
                sstore(buf ^ 1);
                __syncthreads();
                buf ^= 1;
            }
        }
    }
    double *P = part + (int64_t)split * m1 * m2;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int ra = a0 + wm * 32 + mt * 8 + (lane >> 2);
                const int cb = b0 + wn * 32 + nt * 8 + (lane & 3) * 2 + e;
                if (ra < m1 && cb < m2) P[(int64_t)ra * m2 + cb] = acc[mt][nt][e];
            }
}

__global__ void gram_reduce_kernel(const double *__restrict__ part, int nsplit, int m1, int m2, bool sym,
                                   double *__restrict__ G, int64_t ldg) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)m1 * m2) return;
    int ra = (int)(t / m2), cb = (int)(t % m2);
    int sa = ra, sb = cb;
    if (sym && cb < ra) { sa = cb; sb = ra; }  // mirror: exactly symmetric
    double s = 0.0;
    const int64_t stride = (int64_t)m1 * m2;
    for (int q = 0; q < nsplit; ++q) s += part[q * stride + (int64_t)sa * m2 + sb];
    G[(int64_t)ra * ldg + cb] = s;
}

// Out[n x m2] = beta*Cin + alpha*X[n x m1] * B[m1 x m2].  upper != 0: B is upper
// triangular (B[k][c] == 0 for k > c), so column tile c0 only needs k < c0 + TILE
// (the skipped terms are exact zeros: same result).
__global__ void __launch_bounds__(THREADS) gemm_kernel(double alpha, const double *__restrict__ X, int64_t ldx,
                                                       int m1, const double *__restrict__ B, int64_t ldb, int m2,
                                                       double beta, const double *Cin, int64_t ldc, double *Out,
                                                       int64_t ldo, int64_t n, int upper) {
    // column tile fastest: the column tiles of one row tile run together and share its
    // X rows through L2 (one DRAM read of X instead of one per column tile)
    const int nct = (m2 + TILE - 1) / TILE;
    const int64_t r0 = (int64_t)(blockIdx.x / nct) * TILE;
    const int c0 = (int)(blockIdx.x % nct) * TILE;
    if (upper && c0 + TILE < m1) m1 = c0 + TILE;
    __shared__ double Xs[2][TILE][KS + PAD];
    __shared__ double Bs[2][KS][TILE + PAD];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr int PER = KS * TILE / THREADS;
    double rx[PER], rb[PER];
    auto gload = [&](int kb) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + q * THREADS;
            // X tile: 64 rows x 16 k (k fastest)
            const int xr = idx / KS, xk = idx % KS;
            const int64_t row = r0 + xr;
            rx[q] = (row < n && kb + xk < m1) ? __ldg(X + row * ldx + kb + xk) : 0.0;
            // B tile: 16 k x 64 cols (col fastest)
            const int bk = idx / TILE, bc = idx % TILE;
            rb[q] = (kb + bk < m1 && c0 + bc < m2) ? __ldg(B + (int64_t)(kb + bk) * ldb + c0 + bc) : 0.0;
        }
    };
    auto sstore = [&](int buf) {
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int idx = tid + q * THREADS;
            Xs[buf][idx / KS][idx % KS] = rx[q];
            Bs[buf][idx / TILE][idx % TILE] = rb[q];
        }
    };
    gload(0);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int kb = 0; kb < m1; kb += KS) {
        const bool more = kb + KS < m1;
        if (more) gload(kb + KS);
#pragma unroll
        for (int kk = 0; kk < KS / 4; ++kk) {
            double af[4], bf[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) af[mt] = Xs[buf][wm * 32 + mt * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[buf][kk * 4 + (lane & 3)][wn * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
        }
        if (more) {
            sstore(buf ^ 1);
            __syncthreads();
            buf ^= 1;
        }
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t row = r0 + wm * 32 + mt * 8 + (lane >> 2);
                const int cb = c0 + wn * 32 + nt * 8 + (lane & 3) * 2 + e;
                if (row < n && cb < m2) {
                    double v = alpha * acc[mt][nt][e];
                    if (beta != 0.0) v += beta * Cin[row * ldc + cb];
                    Out[row * ldo + cb] = v;
                }
            }
}


// ---------------------------------------------------------------- cp.async pipelined versions
// Same tiles, fragments, DMMA order and reduction as gram_kernel / gemm_kernel (so the
// results are bitwise identical), with the global -> shared copies done by cp.async
// 16-byte chunks into an S-stage ring: S-1 stages in flight while one is computed,
// no staging registers.  Needs 16-byte aligned rows (even ld, even column offsets).
#ifndef ARR_DMMA_STAGES
#define ARR_DMMA_STAGES 2  // measured on B200: 2 stages at 5 CTAs/SM beat 4 stages at 3 (cfg3 ARR basis 623 -> 576 ms)
#endif
#ifndef ARR_DMMA_MINB
// 4 CTAs/SM (128 registers): the A fragments of a k-step get their own registers (at 5 CTAs,
// 96 registers, one register pair was reloaded before every 4 DMMAs); +1-2% on every ARR
// GEMM shape (profiles/r02/dmma_gemm_minb.log)
#define ARR_DMMA_MINB 4
#endif
constexpr int S_CA = ARR_DMMA_STAGES;

__device__ __forceinline__ void ca16(void *smem, const void *gmem, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ca_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ca_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(THREADS, ARR_DMMA_MINB) gram_kernel_ca(const double *__restrict__ X, int64_t ldx, int m1,
                                                          const double *__restrict__ Y, int64_t ldy, int m2,
                                                          int64_t n, int64_t rows_per_split, bool sym,
                                                          double *__restrict__ part) {
    const int ta = blockIdx.x, tb = blockIdx.y, split = blockIdx.z;
    if (sym && tb < ta) return;
    const int a0 = ta * TILE, b0 = tb * TILE;
    const int64_t k0 = (int64_t)split * rows_per_split;
    int64_t k1 = k0 + rows_per_split;
    if (k1 > n) k1 = n;
    extern __shared__ __align__(16) double dsm[];
    double (*Xs)[KS][TILE + PAD] = reinterpret_cast<double (*)[KS][TILE + PAD]>(dsm);
    double (*Ys)[KS][TILE + PAD] = reinterpret_cast<double (*)[KS][TILE + PAD]>(dsm + S_CA * KS * (TILE + PAD));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const bool work = (a0 + wm * 32 < m1) && (b0 + wn * 32 < m2) && !(sym && ta == tb && wm > wn);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // one stage = KS rows x 64 columns of X and of Y = 2 x 512 chunks of 16 bytes, 4 + 4 per thread
    auto load = [&](int64_t kb, int st) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int idx = tid + q * THREADS;
            const int rr = idx >> 5, cc = (idx & 31) * 2;
            const int64_t row = kb + rr;
            const bool rok = row < k1;
            const int nx = rok ? max(0, min(2, m1 - (a0 + cc))) : 0;
            const int ny = rok ? max(0, min(2, m2 - (b0 + cc))) : 0;
            ca16(&Xs[st][rr][cc], nx ? X + row * ldx + a0 + cc : X, nx * 8);
            ca16(&Ys[st][rr][cc], ny ? Y + row * ldy + b0 + cc : Y, ny * 8);
        }
    };
    const int64_t nk = (k1 - k0 + KS - 1) / KS;
#pragma unroll
    for (int st = 0; st < S_CA - 1; ++st) {
        if (st < nk) load(k0 + st * KS, st);
        ca_commit();
    }
    for (int64_t it = 0; it < nk; ++it) {
        ca_wait<S_CA - 2>();
        __syncthreads();
        const int64_t nx = it + S_CA - 1;
        if (nx < nk) load(k0 + nx * KS, (int)(nx % S_CA));
        ca_commit();
        const int buf = (int)(it % S_CA);
        if (work) {
#pragma unroll
            for (int kk = 0; kk < KS / 4; ++kk) {
                double af[4], bf[4];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt) af[mt] = Xs[buf][kk * 4 + (lane & 3)][wm * 32 + mt * 8 + (lane >> 2)];
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) bf[nt] = Ys[buf][kk * 4 + (lane & 3)][wn * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
            }
        }
    }
    ca_wait<0>();
    double *P = part + (int64_t)split * m1 * m2;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int ra = a0 + wm * 32 + mt * 8 + (lane >> 2);
                const int cb = b0 + wn * 32 + nt * 8 + (lane & 3) * 2 + e;
                if (ra < m1 && cb < m2) P[(int64_t)ra * m2 + cb] = acc[mt][nt][e];
            }
}

__global__ void __launch_bounds__(THREADS, ARR_DMMA_MINB) gemm_kernel_ca(double alpha, const double *__restrict__ X, int64_t ldx,
                                                          int m1, const double *__restrict__ B, int64_t ldb, int m2,
                                                          double beta, const double *Cin, int64_t ldc, double *Out,
                                                          int64_t ldo, int64_t n, int upper) {
    // column tile fastest: the column tiles of one row tile run together and share its
    // X rows through L2 (one DRAM read of X instead of one per column tile)
    const int nct = (m2 + TILE - 1) / TILE;
    const int64_t r0 = (int64_t)(blockIdx.x / nct) * TILE;
    const int c0 = (int)(blockIdx.x % nct) * TILE;
    if (upper && c0 + TILE < m1) m1 = c0 + TILE;
    extern __shared__ __align__(16) double dsm[];
    double (*Xs)[TILE][KS + PAD] = reinterpret_cast<double (*)[TILE][KS + PAD]>(dsm);
    double (*Bs)[KS][TILE + PAD] = reinterpret_cast<double (*)[KS][TILE + PAD]>(dsm + S_CA * TILE * (KS + PAD));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // one stage = 64 rows x 16 k of X (8 chunks per row) and 16 k x 64 columns of B (32 chunks per row)
    auto load = [&](int kb, int st) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int idx = tid + q * THREADS;
            const int xr = idx >> 3, xk = (idx & 7) * 2;
            const int64_t row = r0 + xr;
            const int nx = row < n ? max(0, min(2, m1 - (kb + xk))) : 0;
            ca16(&Xs[st][xr][xk], nx ? X + row * ldx + kb + xk : X, nx * 8);
            const int bk = idx >> 5, bc = (idx & 31) * 2;
            const int nb = (kb + bk < m1) ? max(0, min(2, m2 - (c0 + bc))) : 0;
            ca16(&Bs[st][bk][bc], nb ? B + (int64_t)(kb + bk) * ldb + c0 + bc : B, nb * 8);
        }
    };
    const int nk = (m1 + KS - 1) / KS;
#pragma unroll
    for (int st = 0; st < S_CA - 1; ++st) {
        if (st < nk) load(st * KS, st);
        ca_commit();
    }
    for (int it = 0; it < nk; ++it) {
        ca_wait<S_CA - 2>();
        __syncthreads();
        const int nx = it + S_CA - 1;
        if (nx < nk) load(nx * KS, nx % S_CA);
        ca_commit();
        const int buf = it % S_CA;
#pragma unroll
        for (int kk = 0; kk < KS / 4; ++kk) {
            double af[4], bf[4];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt) af[mt] = Xs[buf][wm * 32 + mt * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[buf][kk * 4 + (lane & 3)][wn * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
            for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
        }
    }
    ca_wait<0>();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t row = r0 + wm * 32 + mt * 8 + (lane >> 2);
                const int cb = c0 + wn * 32 + nt * 8 + (lane & 3) * 2 + e;
                if (row < n && cb < m2) {
                    double v = alpha * acc[mt][nt][e];
                    if (beta != 0.0) v += beta * Cin[row * ldc + cb];
                    Out[row * ldo + cb] = v;
                }
            }
}

bool ca_ok(const void *p, int64_t ld) { return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0); }

// ---------------------------------------------------------------- tile-shape variants
// BM x BN CTA tiles of WTM x WTN warp tiles ((WTM/8) x (WTN/8) DMMA m8n8k4 tiles each),
// KSX rows (Gram) / k-columns (GEMM) per stage, an SS-stage cp.async ring (SS - 1 stages in
// flight).  Warp sub-tiles outside the output (or, symmetric, strictly below the diagonal)
// skip their DMMAs.  Same fragments and per-element k order as the 64 x 64 kernels above
// (bitwise the same sums).  Selected with ARRABIT_DMMA_TILE = 1..6 (tuning experiments;
// profiles/r02 logs); 0 = the 64 x 64 kernels above.
constexpr int BPAD = 4;

template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB>
struct DCfg {
    static constexpr int WM = BM / WTM, WN = BN / WTN, THREADS = WM * WN * 32;
    static constexpr int FM = WTM / 8, FN = WTN / 8;
    static constexpr size_t gram_smem = sizeof(double) * SS * KSX * ((BM + BPAD) + (BN + BPAD));
    static constexpr size_t gemm_smem = sizeof(double) * SS * (BM * (KSX + BPAD) + KSX * (BN + BPAD));
};

template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB>
__global__ void __launch_bounds__(DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>::THREADS, MINB)
    gram_kernel_v(const double *__restrict__ X, int64_t ldx, int m1, const double *__restrict__ Y, int64_t ldy,
                  int m2, int64_t n, int64_t rows_per_split, bool sym, double *__restrict__ part) {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    const int ta = blockIdx.x, tb = blockIdx.y, split = blockIdx.z;
    const int a0 = ta * BM, b0 = tb * BN;
    if (sym && b0 + BN <= a0) return;  // strictly below the diagonal
    const int64_t k0 = (int64_t)split * rows_per_split;
    int64_t k1 = k0 + rows_per_split;
    if (k1 > n) k1 = n;
    extern __shared__ __align__(16) double dsm[];
    double (*Xs)[KSX][BM + BPAD] = reinterpret_cast<double (*)[KSX][BM + BPAD]>(dsm);
    double (*Ys)[KSX][BN + BPAD] = reinterpret_cast<double (*)[KSX][BN + BPAD]>(dsm + SS * KSX * (BM + BPAD));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / C::WN, wn = warp % C::WN;
    const int ra0 = a0 + wm * WTM, cb0 = b0 + wn * WTN;
    const bool work = (ra0 < m1) && (cb0 < m2) && !(sym && ra0 >= cb0 + WTN);
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr int CX = KSX * BM / 2, CY = KSX * BN / 2;  // 16-byte chunks per stage
    auto load = [&](int64_t kb, int st) {
#pragma unroll
        for (int idx0 = 0; idx0 < CX + CY; idx0 += C::THREADS) {
            const int idx = idx0 + tid;
            if (idx < CX) {
                const int rr = idx / (BM / 2), cc = (idx % (BM / 2)) * 2;
                const int64_t row = kb + rr;
                const int nx = row < k1 ? max(0, min(2, m1 - (a0 + cc))) : 0;
                ca16(&Xs[st][rr][cc], nx ? X + row * ldx + a0 + cc : X, nx * 8);
            } else if (idx < CX + CY) {
                const int j = idx - CX;
                const int rr = j / (BN / 2), cc = (j % (BN / 2)) * 2;
                const int64_t row = kb + rr;
                const int ny = row < k1 ? max(0, min(2, m2 - (b0 + cc))) : 0;
                ca16(&Ys[st][rr][cc], ny ? Y + row * ldy + b0 + cc : Y, ny * 8);
            }
        }
    };
    const int64_t nk = (k1 - k0 + KSX - 1) / KSX;
#pragma unroll
    for (int st = 0; st < SS - 1; ++st) {
        if (st < nk) load(k0 + st * KSX, st);
        ca_commit();
    }
    for (int64_t it = 0; it < nk; ++it) {
        ca_wait<SS - 2>();
        __syncthreads();
        const int64_t nx = it + SS - 1;
        if (nx < nk) load(k0 + nx * KSX, (int)(nx % SS));
        ca_commit();
        const int buf = (int)(it % SS);
        if (work) {
#pragma unroll
            for (int kk = 0; kk < KSX / 4; ++kk) {
                double af[C::FM], bf[C::FN];
#pragma unroll
                for (int mt = 0; mt < C::FM; ++mt) af[mt] = Xs[buf][kk * 4 + (lane & 3)][wm * WTM + mt * 8 + (lane >> 2)];
#pragma unroll
                for (int nt = 0; nt < C::FN; ++nt) bf[nt] = Ys[buf][kk * 4 + (lane & 3)][wn * WTN + nt * 8 + (lane >> 2)];
#pragma unroll
                for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::FN; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
            }
        }
    }
    ca_wait<0>();
    if (!work) return;
    double *P = part + (int64_t)split * m1 * m2;
#pragma unroll
    for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::FN; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int ra = ra0 + mt * 8 + (lane >> 2);
                const int cb = cb0 + nt * 8 + (lane & 3) * 2 + e;
                if (ra < m1 && cb < m2) P[(int64_t)ra * m2 + cb] = acc[mt][nt][e];
            }
}

template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB>
__global__ void __launch_bounds__(DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>::THREADS, MINB)
    gemm_kernel_v(double alpha, const double *__restrict__ X, int64_t ldx, int m1, const double *__restrict__ B,
                  int64_t ldb, int m2, double beta, const double *Cin, int64_t ldc, double *Out, int64_t ldo,
                  int64_t n, int upper) {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    const int nct = (m2 + BN - 1) / BN;
    const int64_t r0 = (int64_t)(blockIdx.x / nct) * BM;
    const int c0 = (int)(blockIdx.x % nct) * BN;
    if (upper && c0 + BN < m1) m1 = c0 + BN;
    extern __shared__ __align__(16) double dsm[];
    double (*Xs)[BM][KSX + BPAD] = reinterpret_cast<double (*)[BM][KSX + BPAD]>(dsm);
    double (*Bs)[KSX][BN + BPAD] = reinterpret_cast<double (*)[KSX][BN + BPAD]>(dsm + SS * BM * (KSX + BPAD));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / C::WN, wn = warp % C::WN;
    const bool work = (r0 + wm * WTM < n) && (c0 + wn * WTN < m2);
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr int CX = BM * KSX / 2, CB = KSX * BN / 2;
    auto load = [&](int kb, int st) {
#pragma unroll
        for (int idx0 = 0; idx0 < CX + CB; idx0 += C::THREADS) {
            const int idx = idx0 + tid;
            if (idx < CX) {
                const int xr = idx / (KSX / 2), xk = (idx % (KSX / 2)) * 2;
                const int64_t row = r0 + xr;
                const int nx = row < n ? max(0, min(2, m1 - (kb + xk))) : 0;
                ca16(&Xs[st][xr][xk], nx ? X + row * ldx + kb + xk : X, nx * 8);
            } else if (idx < CX + CB) {
                const int j = idx - CX;
                const int bk = j / (BN / 2), bc = (j % (BN / 2)) * 2;
                const int nb = (kb + bk < m1) ? max(0, min(2, m2 - (c0 + bc))) : 0;
                ca16(&Bs[st][bk][bc], nb ? B + (int64_t)(kb + bk) * ldb + c0 + bc : B, nb * 8);
            }
        }
    };
    const int nk = (m1 + KSX - 1) / KSX;
#pragma unroll
    for (int st = 0; st < SS - 1; ++st) {
        if (st < nk) load(st * KSX, st);
        ca_commit();
    }
    for (int it = 0; it < nk; ++it) {
        ca_wait<SS - 2>();
        __syncthreads();
        const int nx = it + SS - 1;
        if (nx < nk) load(nx * KSX, nx % SS);
        ca_commit();
        const int buf = it % SS;
        if (work) {
#pragma unroll
            for (int kk = 0; kk < KSX / 4; ++kk) {
                double af[C::FM], bf[C::FN];
#pragma unroll
                for (int mt = 0; mt < C::FM; ++mt) af[mt] = Xs[buf][wm * WTM + mt * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
#pragma unroll
                for (int nt = 0; nt < C::FN; ++nt) bf[nt] = Bs[buf][kk * 4 + (lane & 3)][wn * WTN + nt * 8 + (lane >> 2)];
#pragma unroll
                for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::FN; ++nt) dmma(acc[mt][nt], af[mt], bf[nt]);
            }
        }
    }
    ca_wait<0>();
    if (!work) return;
#pragma unroll
    for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::FN; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t row = r0 + wm * WTM + mt * 8 + (lane >> 2);
                const int cb = c0 + wn * WTN + nt * 8 + (lane & 3) * 2 + e;
                if (row < n && cb < m2) {
                    double v = alpha * acc[mt][nt][e];
                    if (beta != 0.0) v += beta * Cin[row * ldc + cb];
                    Out[row * ldo + cb] = v;
                }
            }
}

// Software-pipelined versions (the CUTLASS multistage pattern): the fragments of step kk+1
// are loaded from shared memory while the DMMAs of step kk run (two fragment buffers), the
// stage's cp.async copies are spread over its kk steps, and the wait + barrier for the next
// stage sit before the last kk step's DMMAs.  Same fragments, same per-element k order:
// bitwise the same sums as the kernels above.
template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB>
__global__ void __launch_bounds__(DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>::THREADS, MINB)
    gram_kernel_pv(const double *__restrict__ X, int64_t ldx, int m1, const double *__restrict__ Y, int64_t ldy,
                   int m2, int64_t n, int64_t rows_per_split, bool sym, double *__restrict__ part) {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    constexpr int KK = KSX / 4;
    const int ta = blockIdx.x, tb = blockIdx.y, split = blockIdx.z;
    const int a0 = ta * BM, b0 = tb * BN;
    if (sym && b0 + BN <= a0) return;  // strictly below the diagonal
    const int64_t k0 = (int64_t)split * rows_per_split;
    int64_t k1 = k0 + rows_per_split;
    if (k1 > n) k1 = n;
    extern __shared__ __align__(16) double dsm[];
    double (*Xs)[KSX][BM + BPAD] = reinterpret_cast<double (*)[KSX][BM + BPAD]>(dsm);
    double (*Ys)[KSX][BN + BPAD] = reinterpret_cast<double (*)[KSX][BN + BPAD]>(dsm + SS * KSX * (BM + BPAD));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / C::WN, wn = warp % C::WN;
    const int ra0 = a0 + wm * WTM, cb0 = b0 + wn * WTN;
    const bool work = (ra0 < m1) && (cb0 < m2) && !(sym && ra0 >= cb0 + WTN);
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr int CX = KSX * BM / 2, CY = KSX * BN / 2;  // 16-byte chunks per stage
    constexpr int NCH = (CX + CY + C::THREADS - 1) / C::THREADS;  // chunks per thread per stage
    auto load_chunk = [&](int64_t kb, int st, int q) {
        const int idx = q * C::THREADS + tid;
        if (idx < CX) {
            const int rr = idx / (BM / 2), cc = (idx % (BM / 2)) * 2;
            const int64_t row = kb + rr;
            const int nx = row < k1 ? max(0, min(2, m1 - (a0 + cc))) : 0;
            ca16(&Xs[st][rr][cc], nx ? X + row * ldx + a0 + cc : X, nx * 8);
        } else if (idx < CX + CY) {
            const int j = idx - CX;
            const int rr = j / (BN / 2), cc = (j % (BN / 2)) * 2;
            const int64_t row = kb + rr;
            const int ny = row < k1 ? max(0, min(2, m2 - (b0 + cc))) : 0;
            ca16(&Ys[st][rr][cc], ny ? Y + row * ldy + b0 + cc : Y, ny * 8);
        }
    };
    const int64_t nk = (k1 - k0 + KSX - 1) / KSX;
#pragma unroll
    for (int st = 0; st < SS - 1; ++st) {
        if (st < nk)
#pragma unroll
            for (int q = 0; q < NCH; ++q) load_chunk(k0 + st * KSX, st, q);
        ca_commit();
    }
    ca_wait<SS - 2>();
    __syncthreads();
    double af[2][C::FM], bf[2][C::FN];
    auto frag = [&](int buf, int kk, int f) {
#pragma unroll
        for (int mt = 0; mt < C::FM; ++mt) af[f][mt] = Xs[buf][kk * 4 + (lane & 3)][wm * WTM + mt * 8 + (lane >> 2)];
#pragma unroll
        for (int nt = 0; nt < C::FN; ++nt) bf[f][nt] = Ys[buf][kk * 4 + (lane & 3)][wn * WTN + nt * 8 + (lane >> 2)];
    };
    if (nk > 0) frag(0, 0, 0);
    for (int64_t it = 0; it < nk; ++it) {
        const int buf = (int)(it % SS);
        const int64_t nx = it + SS - 1;
        const int nbuf = (int)(nx % SS);
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
            // this stage's share of the copies of stage it + SS - 1 (into the buffer every warp
            // finished reading before the previous barrier)
#pragma unroll
            for (int q = kk; q < NCH; q += KK)
                if (nx < nk) load_chunk(k0 + nx * KSX, nbuf, q);
            if (kk == KK - 1) {
                ca_commit();
                if (it + 1 < nk) {
                    ca_wait<SS - 2>();
                    __syncthreads();
                    frag((int)((it + 1) % SS), 0, (kk + 1) & 1);
                }
            } else {
                frag(buf, kk + 1, (kk + 1) & 1);
            }
            if (work) {
#pragma unroll
                for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::FN; ++nt) dmma(acc[mt][nt], af[kk & 1][mt], bf[kk & 1][nt]);
            }
        }
    }
    ca_wait<0>();
    if (!work) return;
    double *P = part + (int64_t)split * m1 * m2;
#pragma unroll
    for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::FN; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int ra = ra0 + mt * 8 + (lane >> 2);
                const int cb = cb0 + nt * 8 + (lane & 3) * 2 + e;
                if (ra < m1 && cb < m2) P[(int64_t)ra * m2 + cb] = acc[mt][nt][e];
            }
}

template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB>
__global__ void __launch_bounds__(DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>::THREADS, MINB)
    gemm_kernel_pv(double alpha, const double *__restrict__ X, int64_t ldx, int m1, const double *__restrict__ B,
                   int64_t ldb, int m2, double beta, const double *Cin, int64_t ldc, double *Out, int64_t ldo,
                   int64_t n, int upper) {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    constexpr int KK = KSX / 4;
    const int nct = (m2 + BN - 1) / BN;
    const int64_t r0 = (int64_t)(blockIdx.x / nct) * BM;
    const int c0 = (int)(blockIdx.x % nct) * BN;
    if (upper && c0 + BN < m1) m1 = c0 + BN;
    extern __shared__ __align__(16) double dsm[];
    double (*Xs)[BM][KSX + BPAD] = reinterpret_cast<double (*)[BM][KSX + BPAD]>(dsm);
    double (*Bs)[KSX][BN + BPAD] = reinterpret_cast<double (*)[KSX][BN + BPAD]>(dsm + SS * BM * (KSX + BPAD));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / C::WN, wn = warp % C::WN;
    const bool work = (r0 + wm * WTM < n) && (c0 + wn * WTN < m2);
    double acc[C::FM][C::FN][2];
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    constexpr int CX = BM * KSX / 2, CB = KSX * BN / 2;
    constexpr int NCH = (CX + CB + C::THREADS - 1) / C::THREADS;
    auto load_chunk = [&](int kb, int st, int q) {
        const int idx = q * C::THREADS + tid;
        if (idx < CX) {
            const int xr = idx / (KSX / 2), xk = (idx % (KSX / 2)) * 2;
            const int64_t row = r0 + xr;
            const int nx = row < n ? max(0, min(2, m1 - (kb + xk))) : 0;
            ca16(&Xs[st][xr][xk], nx ? X + row * ldx + kb + xk : X, nx * 8);
        } else if (idx < CX + CB) {
            const int j = idx - CX;
            const int bk = j / (BN / 2), bc = (j % (BN / 2)) * 2;
            const int nb = (kb + bk < m1) ? max(0, min(2, m2 - (c0 + bc))) : 0;
            ca16(&Bs[st][bk][bc], nb ? B + (int64_t)(kb + bk) * ldb + c0 + bc : B, nb * 8);
        }
    };
    const int nk = (m1 + KSX - 1) / KSX;
#pragma unroll
    for (int st = 0; st < SS - 1; ++st) {
        if (st < nk)
#pragma unroll
            for (int q = 0; q < NCH; ++q) load_chunk(st * KSX, st, q);
        ca_commit();
    }
    ca_wait<SS - 2>();
    __syncthreads();
    double af[2][C::FM], bf[2][C::FN];
    auto frag = [&](int buf, int kk, int f) {
#pragma unroll
        for (int mt = 0; mt < C::FM; ++mt) af[f][mt] = Xs[buf][wm * WTM + mt * 8 + (lane >> 2)][kk * 4 + (lane & 3)];
#pragma unroll
        for (int nt = 0; nt < C::FN; ++nt) bf[f][nt] = Bs[buf][kk * 4 + (lane & 3)][wn * WTN + nt * 8 + (lane >> 2)];
    };
    if (nk > 0) frag(0, 0, 0);
    for (int it = 0; it < nk; ++it) {
        const int buf = it % SS;
        const int nx = it + SS - 1;
        const int nbuf = nx % SS;
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
#pragma unroll
            for (int q = kk; q < NCH; q += KK)
                if (nx < nk) load_chunk(nx * KSX, nbuf, q);
            if (kk == KK - 1) {
                ca_commit();
                if (it + 1 < nk) {
                    ca_wait<SS - 2>();
                    __syncthreads();
                    frag((it + 1) % SS, 0, (kk + 1) & 1);
                }
            } else {
                frag(buf, kk + 1, (kk + 1) & 1);
            }
            if (work) {
#pragma unroll
                for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
                    for (int nt = 0; nt < C::FN; ++nt) dmma(acc[mt][nt], af[kk & 1][mt], bf[kk & 1][nt]);
            }
        }
    }
    ca_wait<0>();
    if (!work) return;
#pragma unroll
    for (int mt = 0; mt < C::FM; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::FN; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t row = r0 + wm * WTM + mt * 8 + (lane >> 2);
                const int cb = c0 + wn * WTN + nt * 8 + (lane & 3) * 2 + e;
                if (row < n && cb < m2) {
                    double v = alpha * acc[mt][nt][e];
                    if (beta != 0.0) v += beta * Cin[row * ldc + cb];
                    Out[row * ldo + cb] = v;
                }
            }
}

// Tile variant of the GEMMs (ARRABIT_DMMA_TILE, default 0: the 64 x 64 cp.async kernels) and of
// the Grams (ARRABIT_DMMA_GRAM, default 7: 64 x 64, 4 stages, software-pipelined; measured on
// B200 at the ARR shapes: +2-10% over variant 0, profiles/r02/dmma_pipelined_variants.log)
int dmma_tile_choice() {
    static const int t = [] { const char *e = getenv("ARRABIT_DMMA_TILE"); return e ? atoi(e) : 0; }();
    return t;
}
int gram_tile_choice() {
    static const int t = [] {
        const char *e = getenv("ARRABIT_DMMA_GRAM");
        if (e) return atoi(e);
        const char *g = getenv("ARRABIT_DMMA_TILE");
        return g ? atoi(g) : 7;
    }();
    return t;
}

// the variants (BM, BN, WTM, WTN, KSX, SS, MINB)
#define DMMA_VARIANTS(X)                    \
    X(1, 64, 64, 32, 32, 16, 3, 4, false)   \
    X(2, 64, 64, 32, 32, 32, 2, 3, false)   \
    X(3, 64, 128, 32, 64, 16, 3, 2, false)  \
    X(4, 128, 64, 64, 32, 16, 3, 2, false)  \
    X(5, 64, 64, 32, 64, 16, 3, 4, false)   \
    X(6, 64, 64, 64, 32, 16, 3, 4, false)   \
    X(7, 64, 64, 32, 32, 16, 4, 3, true)    \
    X(8, 64, 64, 32, 32, 16, 3, 4, true)    \
    X(9, 64, 128, 32, 64, 16, 3, 2, true)   \
    X(10, 128, 64, 64, 32, 16, 3, 2, true)  \
    X(11, 64, 64, 32, 32, 32, 3, 2, true)   \
    X(12, 128, 128, 32, 64, 16, 3, 1, true) \
    X(13, 128, 64, 32, 32, 16, 3, 2, true)  \
    X(14, 64, 128, 32, 32, 16, 3, 2, true)

struct VarInfo {
    int BM, BN;
    int per_sm;
};

template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB, bool PIPE>
VarInfo var_info() {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    static LaunchCache cache;
    return {BM, BN,
            PIPE ? cached_occupancy(cache, gram_kernel_pv<BM, BN, WTM, WTN, KSX, SS, MINB>, C::THREADS, C::gram_smem)
                 : cached_occupancy(cache, gram_kernel_v<BM, BN, WTM, WTN, KSX, SS, MINB>, C::THREADS, C::gram_smem)};
}
bool variant_info(int v, VarInfo &out) {
    switch (v) {
#define X_INFO(id, a, b, c, d, e, f, g, pipe) \
    case id: out = var_info<a, b, c, d, e, f, g, pipe>(); return true;
        DMMA_VARIANTS(X_INFO)
#undef X_INFO
    }
    return false;
}
template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB, bool PIPE>
void launch_gram_var(arr_ctx *c, const double *X, int64_t ldx, int m1, const double *Y, int64_t ldy, int m2,
                     int64_t n, int64_t rps, int ns, bool sym, double *partials) {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    auto kern = PIPE ? gram_kernel_pv<BM, BN, WTM, WTN, KSX, SS, MINB> : gram_kernel_v<BM, BN, WTM, WTN, KSX, SS, MINB>;
    static LaunchCache cache;
    cached_occupancy(cache, kern, C::THREADS, C::gram_smem);
    dim3 gb((m1 + BM - 1) / BM, (m2 + BN - 1) / BN, ns);
    kern<<<gb, C::THREADS, C::gram_smem, c->stream>>>(X, ldx, m1, Y, ldy, m2, n, rps, sym, partials);
}
template <int BM, int BN, int WTM, int WTN, int KSX, int SS, int MINB, bool PIPE>
void launch_gemm_var(arr_ctx *c, double alpha, const double *X, int64_t ldx, int m1, const double *B, int64_t ldb,
                     int m2, double beta, const double *Cin, int64_t ldc, double *Out, int64_t ldo, int64_t n,
                     int upper) {
    using C = DCfg<BM, BN, WTM, WTN, KSX, SS, MINB>;
    auto kern = PIPE ? gemm_kernel_pv<BM, BN, WTM, WTN, KSX, SS, MINB> : gemm_kernel_v<BM, BN, WTM, WTN, KSX, SS, MINB>;
    static LaunchCache cache;
    cached_occupancy(cache, kern, C::THREADS, C::gemm_smem);
    const unsigned gb = (unsigned)(((n + BM - 1) / BM) * ((m2 + BN - 1) / BN));
    kern<<<gb, C::THREADS, C::gemm_smem, c->stream>>>(alpha, X, ldx, m1, B, ldb, m2, beta, Cin, ldc, Out, ldo, n, upper);
}
bool gram_variant(int v, arr_ctx *c, const double *X, int64_t ldx, int m1, const double *Y, int64_t ldy, int m2,
                  int64_t n, int64_t rps, int ns, bool sym, double *partials) {
    switch (v) {
#define X_GRAM(id, a, b, cc, d, e, f, g, pipe)                                                \
    case id:                                                                                  \
        launch_gram_var<a, b, cc, d, e, f, g, pipe>(c, X, ldx, m1, Y, ldy, m2, n, rps, ns, sym, partials); \
        return true;
        DMMA_VARIANTS(X_GRAM)
#undef X_GRAM
    }
    return false;
}
bool gemm_variant(int v, arr_ctx *c, double alpha, const double *X, int64_t ldx, int m1, const double *B, int64_t ldb,
                  int m2, double beta, const double *Cin, int64_t ldc, double *Out, int64_t ldo, int64_t n,
                  int upper) {
    switch (v) {
#define X_GEMM(id, a, b, cc, d, e, f, g, pipe)                                                                    \
    case id:                                                                                                      \
        launch_gemm_var<a, b, cc, d, e, f, g, pipe>(c, alpha, X, ldx, m1, B, ldb, m2, beta, Cin, ldc, Out, ldo, n, upper); \
        return true;
        DMMA_VARIANTS(X_GEMM)
#undef X_GEMM
    }
    return false;
}

// ---------------------------------------------------------------- small dense
__global__ void svqb_prep_kernel(const double *__restrict__ G, int w, double *__restrict__ D,
                                 double *__restrict__ Gs) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)w * w) return;
    const int i = (int)(t / w), j = (int)(t % w);
    const double gi = G[(int64_t)i * w + i], gj = G[(int64_t)j * w + j];
    const double di = gi > 0.0 ? 1.0 / sqrt(gi) : 0.0;
    const double dj = gj > 0.0 ? 1.0 / sqrt(gj) : 0.0;
    // symmetrise while scaling (G is symmetric up to rounding of the split sums)
    Gs[t] = di * (0.5 * (G[t] + G[(int64_t)j * w + i])) * dj;
    if (j == 0) D[i] = di;
}

__global__ void svqb_build_kernel(const double *__restrict__ D, const double *__restrict__ Vcm,
                                  const double *__restrict__ lam, int w, double tau, double *__restrict__ B,
                                  int *rank_out) {
    const double lmax = lam[w - 1];
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t == 0 && rank_out) {
        int r = 0;
        for (int j = 0; j < w; ++j) r += (lmax > 0.0 && lam[j] > 1e-14 * lmax);
        *rank_out = r;
    }
    if (t >= (int64_t)w * w) return;
    const int i = (int)(t / w), j = (int)(t % w);
    double l = lam[j];
    const double floor_l = tau * lmax;
    if (l < floor_l) l = floor_l;
    B[t] = (lmax > 0.0) ? D[i] * Vcm[(int64_t)j * w + i] / sqrt(l) : 0.0;
}

// H (m x m) was computed by column blocks of width bw, column block J only for
// rows < (J+1)*bw (the upper block triangle).  For i < j: if (j, i) was also
// computed (same diagonal block) average the pair, else mirror (i, j) into (j, i).
__global__ void symmetrize_kernel(double *H, int m, int bw) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)m * m) return;
    const int i = (int)(t / m), j = (int)(t % m);
    if (j <= i) return;
    const bool both = j < (i / bw + 1) * bw;
    const double up = H[(int64_t)i * m + j];
    const double v = both ? 0.5 * (up + H[(int64_t)j * m + i]) : up;
    H[(int64_t)i * m + j] = v;
    H[(int64_t)j * m + i] = v;
}

__global__ void ritz_select_kernel(const double *__restrict__ Vcm, int m, int wsel, double *__restrict__ Vsel) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)m * wsel) return;
    const int i = (int)(t / wsel), j = (int)(t % wsel);
    Vsel[t] = Vcm[(int64_t)(m - 1 - j) * m + i];
}

inline unsigned nblk(int64_t total, int threads) { return (unsigned)((total + threads - 1) / threads); }

}  // namespace

// Row splits of a Gram launch: as many as fill ONE wave of resident CTAs (a
// partial second wave would idle most SMs for a whole CTA lifetime), at least 512
// rows each.  sym: only the upper tiles do work.
int gram_nsplit(int64_t n, int32_t m1, int32_t m2, int num_sms, bool sym) {
    VarInfo vi{TILE, TILE, 0};
    const bool var = gram_tile_choice() > 0 && variant_info(gram_tile_choice(), vi);
    const int TM = vi.BM, TN = vi.BN;
    const int64_t ta = (m1 + TM - 1) / TM, tb = (m2 + TN - 1) / TN;
    // symmetric: tiles on or above the diagonal (tile b intersects columns >= the tile's first row)
    int64_t tiles = ta * tb;
    if (sym) {
        tiles = 0;
        for (int64_t i = 0; i < ta; ++i)
            for (int64_t j = 0; j < tb; ++j) tiles += ((j + 1) * TN > i * TM) ? 1 : 0;
    }
#if ARR_DMMA_CA
    static LaunchCache cache;
    const int per_sm = var ? vi.per_sm
                           : cached_occupancy(cache, gram_kernel_ca, THREADS, sizeof(double) * 2 * S_CA * KS * (TILE + PAD));
#else
    static const int per_sm = [] {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, gram_kernel, THREADS, 0);
        return o > 0 ? o : 1;
    }();
#endif
    const int64_t slots = (int64_t)num_sms * per_sm;
    int64_t ns = slots / tiles;
    if (ns < 1) ns = 1;
    int64_t maxns = n / 512;
    if (maxns > 128) maxns = 128;
    if (maxns < 1) maxns = 1;
    if (ns > maxns) ns = maxns;
    // wave quantisation: tiles*ns CTAs fill ceil(tiles*ns/slots) waves; take the smallest
    // split count from ns up whose last wave is >= 95% full (else the best fill seen)
    auto fill = [&](int64_t q) {
        const double w = (double)(tiles * q) / (double)slots;
        return w / std::ceil(w);
    };
    int64_t best = ns;
    for (int64_t q = ns; q <= maxns; ++q) {
        if (fill(q) > fill(best) + 1e-9) best = q;
        if (fill(best) >= 0.95) break;
    }
    return (int)best;
}

void launch_gram(arr_ctx *c, const double *X, int64_t ldx, int32_t m1, const double *Y, int64_t ldy,
                 int32_t m2, int64_t n, double *G, int64_t ldg, double *partials, bool sym_result) {
    const bool sym = (sym_result || ((X == Y) && (ldx == ldy))) && (m1 == m2);
    int ns = gram_nsplit(n, m1, m2, c->num_sms, sym);
    while ((size_t)ns * m1 * m2 > c->part_elems && ns > 1) --ns;
    int64_t rps = (n + ns - 1) / ns;
    rps = (rps + KS - 1) / KS * KS;
    dim3 grid((m1 + TILE - 1) / TILE, (m2 + TILE - 1) / TILE, ns);
    const int ev0 = t_mark(c);  // the DMMA kernel alone (eig_kernel_times phase 6)
#if ARR_DMMA_CA
    if (gram_tile_choice() > 0 && ca_ok(X, ldx) && ca_ok(Y, ldy) &&
        gram_variant(gram_tile_choice(), c, X, ldx, m1, Y, ldy, m2, n, rps, ns, sym, partials)) {
    } else if (ca_ok(X, ldx) && ca_ok(Y, ldy)) {
        const size_t smem = sizeof(double) * 2 * S_CA * KS * (TILE + PAD);
        static LaunchCache cache;
        cached_occupancy(cache, gram_kernel_ca, THREADS, smem);  // sets the smem attribute once
        gram_kernel_ca<<<grid, THREADS, smem, c->stream>>>(X, ldx, m1, Y, ldy, m2, n, rps, sym, partials);
    } else
#endif
    gram_kernel<<<grid, THREADS, 0, c->stream>>>(X, ldx, m1, Y, ldy, m2, n, rps, sym, partials);
    // algorithmic flops: 2 n m1 m2, the upper triangle n m (m + 1) for a symmetric Gram
    t_add(c, 6, ev0, t_mark(c), 1, sym ? (double)n * m1 * (m1 + 1.0) : 2.0 * n * m1 * m2);
    gram_reduce_kernel<<<nblk((int64_t)m1 * m2, 256), 256, 0, c->stream>>>(partials, ns, m1, m2, sym, G, ldg);
    c->launches += 2;
}

void launch_gemm(arr_ctx *c, double alpha, const double *X, int64_t ldx, int32_t m1, const double *B,
                 int64_t ldb, int32_t m2, double beta, const double *Cin, int64_t ldc, double *Out, int64_t ldo,
                 int64_t n, int upper) {
    const unsigned grid = (unsigned)(((n + TILE - 1) / TILE) * ((m2 + TILE - 1) / TILE));
    const int ev0 = t_mark(c);  // eig_kernel_times phase 7
#if ARR_DMMA_CA
    if (dmma_tile_choice() > 0 && ca_ok(X, ldx) && ca_ok(B, ldb) &&
        gemm_variant(dmma_tile_choice(), c, alpha, X, ldx, m1, B, ldb, m2, beta, Cin, ldc, Out, ldo, n, upper)) {
    } else if (ca_ok(X, ldx) && ca_ok(B, ldb)) {
        const size_t smem = sizeof(double) * S_CA * (TILE * (KS + PAD) + KS * (TILE + PAD));
        static LaunchCache cache;
        cached_occupancy(cache, gemm_kernel_ca, THREADS, smem);  // sets the smem attribute once
        gemm_kernel_ca<<<grid, THREADS, smem, c->stream>>>(alpha, X, ldx, m1, B, ldb, m2, beta, Cin, ldc, Out, ldo, n,
                                                           upper);
    } else
#endif
    gemm_kernel<<<grid, THREADS, 0, c->stream>>>(alpha, X, ldx, m1, B, ldb, m2, beta, Cin, ldc, Out, ldo, n, upper);
    // algorithmic flops: 2 n m1 m2; B upper triangular: 2 n sum_c min(c + 1, m1)
    const double mults = !upper ? (double)m1 * m2
                                : (m2 >= m1 ? 0.5 * m1 * (m1 + 1.0) + (double)(m2 - m1) * m1 : 0.5 * m2 * (m2 + 1.0));
    t_add(c, 7, ev0, t_mark(c), 1, 2.0 * n * mults);
    c->launches++;
}

void launch_svqb_prep(arr_ctx *c, const double *G, int32_t w, double *D, double *Gs) {
    svqb_prep_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(G, w, D, Gs);
    c->launches++;
}

void launch_svqb_build(arr_ctx *c, const double *D, const double *Vcm, const double *lam, int32_t w, double tau,
                       double *B, int *rank_out) {
    svqb_build_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(D, Vcm, lam, w, tau, B, rank_out);
    c->launches++;
}

void launch_symmetrize(arr_ctx *c, double *H, int32_t m, int32_t bw) {
    symmetrize_kernel<<<nblk((int64_t)m * m, 256), 256, 0, c->stream>>>(H, m, bw);
    c->launches++;
}

void launch_ritz_select(arr_ctx *c, const double *Vcm, int32_t m, int32_t wsel, double *Vsel) {
    ritz_select_kernel<<<nblk((int64_t)m * wsel, 256), 256, 0, c->stream>>>(Vcm, m, wsel, Vsel);
    c->launches++;
}

// ---------------------------------------------------------------- CholeskyQR helpers
namespace {
// Gs = D G D + shift*I with D = diag(G)^{-1/2} (column equilibration; 0 for zero columns)
__global__ void chol_prep_kernel(const double *__restrict__ G, int w, double shift, double *__restrict__ D,
                                 double *__restrict__ Gs) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)w * w) return;
    const int i = (int)(t / w), j = (int)(t % w);
    const double gi = G[(int64_t)i * w + i], gj = G[(int64_t)j * w + j];
    const double di = gi > 0.0 ? 1.0 / sqrt(gi) : 0.0;
    const double dj = gj > 0.0 ? 1.0 / sqrt(gj) : 0.0;
    double v = di * (0.5 * (G[t] + G[(int64_t)j * w + i])) * dj;
    if (i == j) v += shift;
    Gs[t] = v;
    if (j == 0) D[i] = di;
}
// B = D * Rinv (row-major), Rinv upper triangular stored column-major (cuSOLVER);
// rank_out (optional) = #{i : R_ii^2 > rank_thr}, read from the factor R kept in Rdiag.
__global__ void chol_build_kernel(const double *__restrict__ D, const double *__restrict__ Rinv_cm, int w,
                                  double *__restrict__ B, const double *__restrict__ Rdiag, double rank_thr,
                                  int *rank_out) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t == 0 && rank_out) {
        int r = 0;
        for (int q = 0; q < w; ++q) r += (Rdiag[q] * Rdiag[q] > rank_thr);
        *rank_out = r;
    }
    if (t >= (int64_t)w * w) return;
    const int i = (int)(t / w), j = (int)(t % w);
    B[t] = (i <= j) ? D[i] * Rinv_cm[(int64_t)j * w + i] : 0.0;
}
__global__ void chol_racc_kernel(const double *__restrict__ Rs_cm, const double *__restrict__ D, int w,
                                 const double *__restrict__ Rold, double *__restrict__ Rnew, bool first) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)w * w) return;
    const int i = (int)(t / w), j = (int)(t % w);
    double v = 0.0;
    if (i <= j) {
        if (first) {
            v = Rs_cm[(int64_t)j * w + i] / D[j];
        } else {
            for (int k = i; k <= j; ++k) v += Rs_cm[(int64_t)k * w + i] / D[k] * Rold[(int64_t)k * w + j];
        }
    }
    Rnew[t] = v;
}
__global__ void put_rt_kernel(const double *__restrict__ R, int w, double *__restrict__ H, int64_t ldh) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)w * w) return;
    const int a = (int)(t / w), b = (int)(t % w);
    H[(int64_t)a * ldh + b] = R[(int64_t)b * w + a];
}
__global__ void diag_copy_kernel(const double *__restrict__ A_cm, int w, double *__restrict__ d) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < w) d[i] = A_cm[(int64_t)i * w + i];
}
}  // namespace

namespace {
// out = max over the upper triangle of |M_ij - delta_ij| (M column-major w x w), one CTA
// out = max_{i <= j} |M(i, j) - delta_ij| (M column-major, upper triangle); NaN wins.
// One CTA per column; the CTA maxima are combined with an integer atomicMax on the
// IEEE bits (order-preserving for non-negative doubles, NaN above +inf): the max is
// order independent, so the result is deterministic.  *out must be zeroed first.
__global__ void dev_from_identity_kernel(const double *__restrict__ M_cm, int w, double *out) {
    const int j = blockIdx.x;
    double m = 0.0;
    for (int i = threadIdx.x; i <= j; i += blockDim.x) {
        const double v = fabs(M_cm[(int64_t)j * w + i] - (i == j ? 1.0 : 0.0));
        m = (v > m || v != v) ? v : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, m, o);
        m = (v > m || v != v) ? v : m;
    }
    if ((threadIdx.x & 31) == 0) {
        const double a = m != m ? __longlong_as_double(0x7ff8000000000000ll) : m;
        atomicMax(reinterpret_cast<unsigned long long *>(out), (unsigned long long)__double_as_longlong(a));
    }
}
}  // namespace

namespace {
// out = max |x_i| over count elements (NaN wins); integer atomicMax on the IEEE bits
// (order-preserving for non-negative doubles): deterministic.  *out zeroed first.
__global__ void maxabs_kernel(const double *__restrict__ x, int64_t count, double *out) {
    double m = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
        const double v = fabs(x[t]);
        m = (v > m || v != v) ? v : m;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double v = __shfl_xor_sync(0xffffffffu, m, o);
        m = (v > m || v != v) ? v : m;
    }
    if ((threadIdx.x & 31) == 0) {
        const double a = m != m ? __longlong_as_double(0x7ff8000000000000ll) : m;
        atomicMax(reinterpret_cast<unsigned long long *>(out), (unsigned long long)__double_as_longlong(a));
    }
}
}  // namespace

namespace {
// M (row-major w x w): M[j][i] = M[i][j] for i < j, then M[i][i] += add_diag
__global__ void mirror_upper_kernel(double *M, int w, double add_diag) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)w * w) return;
    const int i = (int)(t / w), j = (int)(t % w);
    if (i < j) M[(int64_t)j * w + i] = M[(int64_t)i * w + j];
    else if (i == j) M[t] += add_diag;
}
__global__ void add_diag_kernel(double *M, int w, int64_t ld, double v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < w) M[(int64_t)i * ld + i] += v;
}
}  // namespace

void launch_mirror_upper(arr_ctx *c, double *M, int32_t w) {
    mirror_upper_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(M, w, 0.0);
    c->launches++;
}
void launch_add_diag(arr_ctx *c, double *M, int32_t w, int64_t ld, double v) {
    add_diag_kernel<<<(w + 255) / 256, 256, 0, c->stream>>>(M, w, ld, v);
    c->launches++;
}

void launch_maxabs(arr_ctx *c, const double *x, int64_t count, double *out) {
    cudaMemsetAsync(out, 0, sizeof(double), c->stream);
    int64_t blocks = (count + 255) / 256;
    if (blocks > (int64_t)c->num_sms * 4) blocks = (int64_t)c->num_sms * 4;
    if (blocks < 1) blocks = 1;
    maxabs_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(x, count, out);
    c->launches++;
}

void launch_dev_from_identity(arr_ctx *c, const double *M_cm, int32_t w, double *out) {
    cudaMemsetAsync(out, 0, sizeof(double), c->stream);
    dev_from_identity_kernel<<<w, 64, 0, c->stream>>>(M_cm, w, out);
    c->launches++;
}

void launch_chol_prep(arr_ctx *c, const double *G, int32_t w, double shift, double *D, double *Gs) {
    chol_prep_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(G, w, shift, D, Gs);
    c->launches++;
}
void launch_chol_build(arr_ctx *c, const double *D, const double *Rinv_cm, int32_t w, double *B, const double *Rdiag,
                       double rank_thr, int *rank_out) {
    chol_build_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(D, Rinv_cm, w, B, Rdiag, rank_thr, rank_out);
    c->launches++;
}
void launch_chol_racc(arr_ctx *c, const double *Rs_cm, const double *D, int32_t w, const double *Rold, double *Rnew,
                      bool first) {
    chol_racc_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(Rs_cm, D, w, Rold, Rnew, first);
    c->launches++;
}
void launch_put_rt(arr_ctx *c, const double *R, int32_t w, double *H, int64_t ldh) {
    put_rt_kernel<<<nblk((int64_t)w * w, 256), 256, 0, c->stream>>>(R, w, H, ldh);
    c->launches++;
}
void launch_diag_copy(arr_ctx *c, const double *A_cm, int32_t w, double *d) {
    diag_copy_kernel<<<nblk(w, 256), 256, 0, c->stream>>>(A_cm, w, d);
    c->launches++;
}
