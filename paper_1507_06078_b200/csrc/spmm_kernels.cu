// Fused CSR x row-major-block kernels for sm_100a: the Chebyshev filter degree
// (Eq. cheby-poly P:377-383 on the map of Eq. rhod, Alg. Arrabit2
// line P:1486), the augmentation SpMM (Alg. ARR) and the residual pass
// (Eq. resi).  HBM-bound: every degree reads A once,
// gathers Y_j rows through L1/L2, streams Y_{j-1} in and Y_{j+1} out with
// evict-first hints, and optionally emits deterministic column sums of squares.
#include <math.h>

#include "internal.cuh"

namespace {

#ifndef ARR_SPMM_MAXT
#define ARR_SPMM_MAXT 512
#endif
#ifndef ARR_SPMM_MINB
#define ARR_SPMM_MINB 2
#endif
#ifndef ARR_SPMM_PAIR
#define ARR_SPMM_PAIR 0
#endif
#ifndef ARR_SPMM_V4
#define ARR_SPMM_V4 0  // 1: 256-bit accesses when the block is 32-byte aligned with ld % 4 == 0
#endif
#ifndef ARR_SPMM_WS
#define ARR_SPMM_WS 1  // warp-specialised kernel: a producer warp stages the CSR of the next tile (2-stage ring)
#endif
#ifndef ARR_SPMM_PF
#define ARR_SPMM_PF 1  // per-thread L2 prefetch of a later row's DRAM-bound operands (Y_{j-1} row, leading-edge gather)
#endif
#ifndef ARR_SPMM_PF_AHEAD
#define ARR_SPMM_PF_AHEAD 2  // rows ahead (cfg2: 107 -> 103 us per degree with 32-row tiles)
#endif
#ifndef ARR_SPMM_SEQ
#define ARR_SPMM_SEQ 0  // 1: each row slot walks a contiguous run of the tile's rows (L1 reuse of x-neighbours)
#endif
constexpr int kMaxThreads = ARR_SPMM_MAXT;  // fused SpMM CTA size (R x TX rounded to warps)

#ifndef ARR_L2HINT
#define ARR_L2HINT 1  // L2 eviction-priority hints: gathers evict_last, streams evict_first
#endif

// Cache-policy handles (createpolicy) and hinted 64/128-bit accesses.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

#if ARR_L2HINT
#define GATHER(p) V::ldg_h((p), pol_keep)
#define STREAM_LD(p) V::ldcs_h((p), pol_stream)
#define STREAM_ST(p, v) V::stcs_h((p), (v), pol_stream)
#else
#define GATHER(p) V::ldg(p)
#define STREAM_LD(p) V::ldcs(p)
#define STREAM_ST(p, v) V::stcs((p), (v))
#endif

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
    using T = double;
    static __device__ __forceinline__ T zero() { return 0.0; }
    static __device__ __forceinline__ T ldg(const double *p) { return __ldg(p); }
    static __device__ __forceinline__ T ldcs(const double *p) { return __ldcs(p); }
    static __device__ __forceinline__ void stcs(double *p, T v) { __stcs(p, v); }
    static __device__ __forceinline__ T ldg_h(const double *p, uint64_t pol) {
        double r;
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
        return r;
    }
    static __device__ __forceinline__ T ldcs_h(const double *p, uint64_t pol) {
        double r;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
        return r;
    }
    static __device__ __forceinline__ void stcs_h(double *p, T v, uint64_t pol) {
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
    }
    static __device__ __forceinline__ double get(const T &v, int) { return v; }
    static __device__ __forceinline__ void set(T &v, int, double x) { v = x; }
};
template <>
struct Vec<2> {
    using T = double2;
    static __device__ __forceinline__ T zero() { return make_double2(0.0, 0.0); }
    static __device__ __forceinline__ T ldg(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }
    static __device__ __forceinline__ T ldcs(const double *p) { return __ldcs(reinterpret_cast<const double2 *>(p)); }
    static __device__ __forceinline__ void stcs(double *p, T v) { __stcs(reinterpret_cast<double2 *>(p), v); }
    static __device__ __forceinline__ T ldg_h(const double *p, uint64_t pol) {
        double2 r;
        asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
        return r;
    }
    static __device__ __forceinline__ T ldcs_h(const double *p, uint64_t pol) {
        double2 r;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                     : "=d"(r.x), "=d"(r.y)
                     : "l"(p), "l"(pol));
        return r;
    }
    static __device__ __forceinline__ void stcs_h(double *p, T v, uint64_t pol) {
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x),
                     "d"(v.y), "l"(pol)
                     : "memory");
    }
    static __device__ __forceinline__ double get(const T &v, int e) { return e ? v.y : v.x; }
    static __device__ __forceinline__ void set(T &v, int e, double x) {
        if (e) v.y = x; else v.x = x;
    }
};

struct __align__(32) d4 {
    double x, y, z, w;
};
template <>
struct Vec<4> {  // 256-bit accesses (sm_100: LDG/STG .ENL2.256)
    using T = d4;
    static __device__ __forceinline__ T zero() { return d4{0.0, 0.0, 0.0, 0.0}; }
    static __device__ __forceinline__ T ldg(const double *p) {
        d4 r;
        asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
        return r;
    }
    static __device__ __forceinline__ T ldcs(const double *p) {
        d4 r;
        asm volatile("ld.global.cs.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w) : "l"(p));
        return r;
    }
    static __device__ __forceinline__ void stcs(double *p, T v) {
        asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                     : "memory");
    }
    static __device__ __forceinline__ T ldg_h(const double *p, uint64_t pol) {
        d4 r;
        asm("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
            : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
            : "l"(p), "l"(pol));
        return r;
    }
    static __device__ __forceinline__ T ldcs_h(const double *p, uint64_t pol) {
        d4 r;
        asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(r.x), "=d"(r.y), "=d"(r.z), "=d"(r.w)
                     : "l"(p), "l"(pol));
        return r;
    }
    static __device__ __forceinline__ void stcs_h(double *p, T v, uint64_t pol) {
        asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p),
                     "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w), "l"(pol)
                     : "memory");
    }
    static __device__ __forceinline__ double get(const T &v, int e) {
        return e == 0 ? v.x : (e == 1 ? v.y : (e == 2 ? v.z : v.w));
    }
    static __device__ __forceinline__ void set(T &v, int e, double x) {
        if (e == 0) v.x = x; else if (e == 1) v.y = x; else if (e == 2) v.z = x; else v.w = x;
    }
};

template <int VEC>
__device__ __forceinline__ void fma_vec(typename Vec<VEC>::T &acc, double a, const typename Vec<VEC>::T &x);
template <>
__device__ __forceinline__ void fma_vec<1>(double &acc, double a, const double &x) { acc = fma(a, x, acc); }
template <>
__device__ __forceinline__ void fma_vec<2>(double2 &acc, double a, const double2 &x) {
    acc.x = fma(a, x.x, acc.x);
    acc.y = fma(a, x.y, acc.y);
}
template <>
__device__ __forceinline__ void fma_vec<4>(d4 &acc, double a, const d4 &x) {
    acc.x = fma(a, x.x, acc.x);
    acc.y = fma(a, x.y, acc.y);
    acc.z = fma(a, x.z, acc.z);
    acc.w = fma(a, x.w, acc.w);
}

constexpr int kTile = 64;  // rows per tile (the unit of the processing order)


// One staged non-zero: element offset of the referenced Y row and the value.
struct __align__(16) Ent {
    int64_t off;  // col * ld_in
    double val;
};

// alpha (acc - shift y_i) with the contraction spelled out (the stencil path,
// stencil_kernels.cu, uses the same sequence: bitwise equal outputs)
__device__ __forceinline__ double epi(double alpha, double acc, double shift, double yi) {
    return alpha * fma(-shift, yi, acc);
}

// Epilogue of one row: out = alpha*(acc - shift*y_i) + beta*y_prev, column
// sums of squares, evict-first store.
template <int VEC, int NV, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
__device__ __forceinline__ void row_epilogue(const SpmmArgs &a, int64_t i, int TX, int v0, int wv,
                                             const typename Vec<VEC>::T (&acc)[NV],
                                             const typename Vec<VEC>::T (&yp)[NV], double (&ss)[NV][VEC],
                                             uint64_t pol_stream) {
    using V = Vec<VEC>;
    using T = typename V::T;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int vv = v0 + v * TX;
        if (vv >= wv) continue;
        const T yi = V::ldg(a.Yin + i * a.ld_in + vv * VEC);
        const T xa = HAS_X ? STREAM_LD(a.Xa + i * a.ld_xa + vv * VEC) : V::zero();
        T out;
#pragma unroll
        for (int e = 0; e < VEC; ++e) {
            const double sh = COLSHIFT ? __ldg(a.colshift + vv * VEC + e) : a.shift;
            double o = epi(a.alpha, V::get(acc[v], e), sh, V::get(yi, e));
            if (HAS_PREV) o = fma(a.scale_mode == 2 ? a.beta * __ldg(a.colscale + vv * VEC + e) : a.beta, V::get(yp[v], e), o);
            if (HAS_X) o = fma(a.gxa, V::get(xa, e), o);
            if (a.scale_mode == 1) o *= __ldg(a.colscale + vv * VEC + e);
            V::set(out, e, o);
            if (SUMSQ) ss[v][e] = fma(o, o, ss[v][e]);
        }
        if (STORE) STREAM_ST(a.Yout + i * a.ld_out + vv * VEC, out);
    }
}

// Rows of one tile owned by row slot r.  Each row is processed in chunks of K
// non-zeros: the K row offsets come from shared memory, the K gathers of Y_j
// are issued back to back (all in flight together), then the values are read
// from shared memory and K FMAs run in CSR order.  Slots past the row end
// re-gather the row's first entry with value 0 (no branches).  When every row
// fits one chunk (K >= longest row) two rows are kept in flight per thread.
template <int VEC, int NV, int K, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
__device__ __forceinline__ void tile_rows(const SpmmArgs &a, int64_t r0, int nrows, int R, int RR, int r, int TX,
                                          int v0, int wv, const int *s_rp, const Ent *s_ent,
                                          double (&ss)[NV][VEC], uint64_t pol_keep, uint64_t pol_stream) {
    using V = Vec<VEC>;
    using T = typename V::T;
    constexpr int P = (ARR_SPMM_PAIR && NV == 1 && K <= 7) ? 2 : 1;  // rows in flight per thread
    RR = (nrows + R - 1) / R;  // rows per slot for this (pass of the) tile
    const double *yin_v[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const int vv = v0 + v * TX;
        yin_v[v] = a.Yin + (vv < wv ? vv : 0) * VEC;
    }
    if constexpr (P == 2) {
        for (int rr = 0; rr < RR; rr += 2) {
            const int lr0 = ARR_SPMM_SEQ ? r * RR + rr : rr * R + r;
            const int lr1 = ARR_SPMM_SEQ ? lr0 + 1 : lr0 + R;
            if (lr0 >= nrows) break;
            const bool has1 = (rr + 1 < RR) && (lr1 < nrows);
            const int64_t i0 = r0 + lr0, i1 = r0 + (has1 ? lr1 : lr0);
            T yp0[NV], yp1[NV];
            if (HAS_PREV) {
                yp0[0] = STREAM_LD(a.Yprev + i0 * a.ld_prev + v0 * VEC);
                yp1[0] = has1 ? STREAM_LD(a.Yprev + i1 * a.ld_prev + v0 * VEC) : V::zero();
            }
            const int p00 = s_rp[lr0], p01 = s_rp[lr0 + 1];
            const int p10 = has1 ? s_rp[lr1] : p01, p11 = has1 ? s_rp[lr1 + 1] : p01;
            const int64_t safe0 = p00 < p01 ? s_ent[p00].off : i0 * a.ld_in;
            const int64_t safe1 = p10 < p11 ? s_ent[p10].off : i1 * a.ld_in;
            T x0[K], x1[K];
#pragma unroll
            for (int u = 0; u < K; ++u) {
                const int64_t o0 = (p00 + u < p01) ? s_ent[p00 + u].off : safe0;
                const int64_t o1 = (p10 + u < p11) ? s_ent[p10 + u].off : safe1;
                x0[u] = GATHER(yin_v[0] + o0);
                x1[u] = GATHER(yin_v[0] + o1);
            }
            T acc0[NV], acc1[NV];
            acc0[0] = V::zero();
            acc1[0] = V::zero();
#pragma unroll
            for (int u = 0; u < K; ++u) {
                const double a0 = (p00 + u < p01) ? s_ent[p00 + u].val : 0.0;
                const double a1 = (p10 + u < p11) ? s_ent[p10 + u].val : 0.0;
                fma_vec<VEC>(acc0[0], a0, x0[u]);
                fma_vec<VEC>(acc1[0], a1, x1[u]);
            }
            if (v0 < wv) {
                row_epilogue<VEC, NV, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>(a, i0, TX, v0, wv, acc0, yp0, ss, pol_stream);
                if (has1) row_epilogue<VEC, NV, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>(a, i1, TX, v0, wv, acc1, yp1, ss, pol_stream);
            }
        }
    } else {
        for (int rr = 0; rr < RR; ++rr) {
            const int lr = ARR_SPMM_SEQ ? r * RR + rr : rr * R + r;
            if (lr >= nrows) break;
            const int64_t i = r0 + lr;
#if ARR_SPMM_PF
            {
                // Only two of a row's loads miss L2 (the Y_{j-1} row and the first touch of
                // its leading-edge gather); pull a later row's into L2 now, without registers.
                const int rn = rr + ARR_SPMM_PF_AHEAD;
                const int lrn = ARR_SPMM_SEQ ? r * RR + rn : rn * R + r;
                if (rn < RR && lrn < nrows) {
                    const int64_t in = r0 + lrn;
                    if (HAS_PREV)
                        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(a.Yprev + in * a.ld_prev + v0 * VEC));
                    const int q1 = s_rp[lrn + 1];
                    if (q1 > s_rp[lrn])
                        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(yin_v[0] + s_ent[q1 - 1].off));
                }
            }
#endif
            T yp[NV];
            if (HAS_PREV) {
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int vv = v0 + v * TX;
                    yp[v] = (vv < wv) ? STREAM_LD(a.Yprev + i * a.ld_prev + vv * VEC) : V::zero();
                }
            }
            const int p0 = s_rp[lr];
            const int p1 = s_rp[lr + 1];
            ARR_CHECK(lr + 1 <= kTile + 1 && p0 >= 0 && p0 <= p1);
            T acc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = V::zero();
            for (int p = p0; p < p1; p += K) {
                T x[K][NV];
                const int64_t safe = s_ent[p].off;
#pragma unroll
                for (int u = 0; u < K; ++u) {
                    ARR_CHECK(p + u < p1 || p >= 0);
                    const int64_t o = (p + u < p1) ? s_ent[p + u].off : safe;
#pragma unroll
                    for (int v = 0; v < NV; ++v) x[u][v] = GATHER(yin_v[v] + o);
                }
#pragma unroll
                for (int u = 0; u < K; ++u) {
                    const double av = (p + u < p1) ? s_ent[p + u].val : 0.0;
#pragma unroll
                    for (int v = 0; v < NV; ++v) fma_vec<VEC>(acc[v], av, x[u][v]);
                }
            }
            row_epilogue<VEC, NV, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>(a, i, TX, v0, wv, acc, yp, ss, pol_stream);
        }
    }
}

// Tiled fused SpMM.  A CTA of R x TX threads (rounded up to whole warps)
// processes tiles of RT = R*RR consecutive rows.  Each tile's CSR slice is
// staged in shared memory with coalesced loads as 16-byte {col*ld, val}
// entries, so the only global latency left per row is the batch of Y_j
// gathers (the row_ptr -> col -> Y chain of a plain CSR loop is paid once per
// tile).  Thread (r, v0) owns row slot r (rows r0 + rr*R + r) and the 16-byte
// column vectors v0, v0+TX, ... (NV of them); Y_{j-1} is prefetched with an
// evict-first load before the gathers and Y_{j+1} is stored evict-first.
// Tiles are visited grid-stride so the rows in flight chip-wide form one
// contiguous window (L2 reuse of gathered neighbour rows).  Per-row sums run
// in CSR order, so results do not depend on the partition or the tiling.
// A tile whose slice exceeds the staging capacity is staged in several passes
// of whole rows.
template <int VEC, int NV, int K, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
__global__ void __launch_bounds__(kMaxThreads, ARR_SPMM_MINB) spmm_tile_kernel(SpmmArgs a, int TX, int R, int RT, int wv,
                                                                    int64_t ntiles, int nnz_cap) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int RR = 0;  // recomputed per tile in tile_rows
    Ent *s_ent = reinterpret_cast<Ent *>(smem_raw);                      // [nnz_cap]
    int *s_rp = reinterpret_cast<int *>(smem_raw + sizeof(Ent) * nnz_cap);  // [kTile+2] (relative)
    __shared__ int64_t s_base;

    const int tid = threadIdx.x;
    const int nthr = blockDim.x;
    const int r = tid / TX;
    const int v0 = tid - r * TX;
    const bool active = r < R;
    double ss[NV][VEC];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < VEC; ++e) ss[v][e] = 0.0;
    const int64_t *__restrict__ rp = a.row_ptr;
    const int32_t *__restrict__ col = a.col;
    const double *__restrict__ val = a.val;
    const int64_t ld = a.ld_in;
    const uint64_t pol_keep = policy_evict_last();
    const uint64_t pol_stream = policy_evict_first();

    // Tile order: launches without a column reduction hand tiles out in order
    // from an atomic ticket (CTAs cannot drift apart, so the rows in flight stay
    // one contiguous window); SUMSQ launches keep the static grid-stride
    // assignment so their per-CTA partial sums are deterministic.
    constexpr bool DYN = !SUMSQ;
    __shared__ int64_t s_next[2];
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; ++it) {
        // next tile of this CTA, taken one tile ahead (read after the staging barriers)
        if (tid == 0) s_next[it & 1] = DYN ? (int64_t)gridDim.x + (int64_t)atomicAdd(a.sched, 1ull) : t + gridDim.x;
        int64_t r0;
        int nrows;
        if (a.tile_row0) {  // caller-given processing order of contiguous row ranges
            r0 = a.tile_row0[t];
            nrows = a.tile_len[t];
        } else {
            r0 = t * RT;
            nrows = (int)min((int64_t)RT, a.n - r0);
        }
        int done = 0;  // rows of this tile already processed
        while (done < nrows) {
            __syncthreads();  // previous pass finished with the staged slice
            if (tid == 0) s_base = __ldg(rp + r0 + done);
            __syncthreads();
            const int64_t base = s_base;
            // rows [done, done+cnt) whose slice fits the capacity (at least one row)
            for (int q = tid; q <= nrows - done; q += nthr) {
                const int64_t o = __ldg(rp + r0 + done + q) - base;
                s_rp[q] = o <= nnz_cap ? (int)o : nnz_cap + 1;
            }
            __syncthreads();
            int cnt = 0;
            {
                // largest cnt with s_rp[cnt] <= nnz_cap (s_rp is nondecreasing)
                int lo = 1, hi = nrows - done;
                if (s_rp[1] > nnz_cap) hi = 0;
                while (lo <= hi) {
                    const int mid = (lo + hi) >> 1;
                    if (s_rp[mid] <= nnz_cap) { cnt = mid; lo = mid + 1; } else hi = mid - 1;
                }
            }
            if (cnt == 0) {
                // a single row longer than the capacity: process it in K-chunks from global memory
                if (active && r == 0) {
                    const int64_t i = r0 + done;
                    using V = Vec<VEC>;
                    using T = typename V::T;
                    const int64_t p0 = __ldg(rp + i), p1 = __ldg(rp + i + 1);
                    for (int v = 0; v < NV; ++v) {
                        const int vv = v0 + v * TX;
                        if (vv >= wv) continue;
                        T acc = V::zero();
                        for (int64_t p = p0; p < p1; ++p)
                            fma_vec<VEC>(acc, __ldg(val + p), V::ldg(a.Yin + (int64_t)__ldg(col + p) * ld + vv * VEC));
                        const T yi = V::ldg(a.Yin + i * ld + vv * VEC);
                        T yp = V::zero();
                        if (HAS_PREV) yp = V::ldcs(a.Yprev + i * a.ld_prev + vv * VEC);
                        T out;
                        for (int e = 0; e < VEC; ++e) {
                            const double sh = COLSHIFT ? __ldg(a.colshift + vv * VEC + e) : a.shift;
                            double o = epi(a.alpha, V::get(acc, e), sh, V::get(yi, e));
                            if (HAS_PREV)
                                o = fma(a.scale_mode == 2 ? a.beta * __ldg(a.colscale + vv * VEC + e) : a.beta,
                                        V::get(yp, e), o);
                            if (HAS_X) o = fma(a.gxa, a.Xa[i * a.ld_xa + vv * VEC + e], o);
                            if (a.scale_mode == 1) o *= __ldg(a.colscale + vv * VEC + e);
                            V::set(out, e, o);
                            if (SUMSQ) ss[v][e] = fma(o, o, ss[v][e]);
                        }
                        if (STORE) V::stcs(a.Yout + i * a.ld_out + vv * VEC, out);
                    }
                }
                // other row-slot threads of the block stay idle for this row
                done += 1;
                continue;
            }
            const int nnz_t = s_rp[cnt];
            for (int q = tid; q < nnz_t; q += nthr) {
                Ent e;
                e.off = (int64_t)__ldg(col + base + q) * ld;
                e.val = __ldg(val + base + q);
                s_ent[q] = e;
            }
            __syncthreads();
            if (active)
                tile_rows<VEC, NV, K, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>(a, r0 + done, cnt, R, RR, r, TX, v0, wv,
                                                                        s_rp, s_ent, ss, pol_keep, pol_stream);
            done += cnt;
        }
        __syncthreads();  // every thread is done with this tile's staging and has s_next
        t = s_next[it & 1];
    }
    if (DYN && tid == 0) {
        // the last CTA to finish resets the ticket for the next launch
        __threadfence();
        if (atomicAdd(a.sched + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
            a.sched[0] = 0;
            a.sched[1] = 0;
            __threadfence();
        }
    }
    if (SUMSQ) {
        // fixed-order block reduction over the R row slots of each column
        double *red = reinterpret_cast<double *>(smem_raw);
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            __syncthreads();
            if (active) {
#pragma unroll
                for (int e = 0; e < VEC; ++e) red[(r * TX + v0) * VEC + e] = ss[v][e];
            }
            __syncthreads();
            const int vv = v0 + v * TX;
            if (active && r == 0 && vv < wv) {
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    double sum = 0.0;
                    for (int q = 0; q < R; ++q) sum += red[(q * TX + v0) * VEC + e];
                    const int colid = vv * VEC + e;
                    if (colid < a.w) a.partials[(int64_t)blockIdx.x * a.w + colid] = sum;
                }
            }
        }
    }
}

#ifndef ARR_SPMM_CAP
#define ARR_SPMM_CAP 2048
#endif
constexpr int kNnzCap = ARR_SPMM_CAP;  // staged CSR entries per tile pass
#ifndef ARR_SPMM_WS_CAP
#define ARR_SPMM_WS_CAP 1792
#endif
constexpr int kWsCap = ARR_SPMM_WS_CAP;  // entries per stage of the warp-specialised kernel (2 stages)

// ---------------------------------------------------------------- warp-specialised tiles
// Named barriers (bar.sync / bar.arrive with a thread count): FULL[s] (ids 1,2)
// and EMPTY[s] (ids 3,4) of the two shared-memory stages.
__device__ __forceinline__ void nb_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void nb_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct WsInfo {
    int64_t r0;  // first row (-1: no more work)
    int nrows;   // rows of this item
    int mode;    // 0: staged slice, 1: one row longer than the stage (read from global memory)
};

// Same arithmetic and per-row CSR order as spmm_tile_kernel.  The last warp is a
// producer: it takes this CTA's tiles in order (atomic ticket, or the static
// grid-stride order for launches that reduce column norms), splits a tile whose
// slice exceeds the stage capacity into row ranges that fit, and stages each
// range's row pointers and {col*ld, val} entries into one of two shared-memory
// stages while the consumer warps compute the other: the CSR round trips of the
// next tile are hidden behind the current one.
template <int VEC, int NV, int K, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
#ifndef ARR_SPMM_WS_MINB
#define ARR_SPMM_WS_MINB 2
#endif
__global__ void __launch_bounds__(kMaxThreads + 32, ARR_SPMM_WS_MINB) spmm_ws_kernel(SpmmArgs a, int TX, int R, int RT, int wv,
                                                                      int64_t ntiles, int nnz_cap, int ncons) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const size_t stage_bytes = ((sizeof(Ent) * (size_t)nnz_cap + 4 * (size_t)(kTile + 2) + 15) & ~size_t(15));
    __shared__ WsInfo s_info[2];
    const int tid = threadIdx.x;
    const int nall = ncons + 32;
    const bool producer = tid >= ncons;
    const int64_t *__restrict__ rp = a.row_ptr;
    const int64_t ld = a.ld_in;
    if (producer) {
        const int lane = tid - ncons;
        int st = 0, k = 0;
        // Stage rows [r0, r0 + nrows) (their CSR slice fits) into stage st: the row
        // pointers were already loaded by the lanes (rpv[h] = rp[r0 + lane + 32h] - base).
        auto wait_stage = [&]() {
            if (k >= 2) nb_sync(3 + st, nall);  // consumers released this stage
        };
        auto release = [&](int64_t r0, int nrows, int mode) {
            if (lane == 0) s_info[st] = WsInfo{r0, nrows, mode};
            __syncwarp();
            nb_arrive(1 + st, nall);
            st ^= 1;
            ++k;
        };
        constexpr bool DYN = !SUMSQ;
        constexpr int UN = 8;  // entries in flight per lane
        for (int64_t t = blockIdx.x; t < ntiles;) {
            int64_t r0;
            int nrows;
            if (a.tile_row0) { r0 = __ldg(a.tile_row0 + t); nrows = __ldg(a.tile_len + t); }
            else { r0 = t * RT; nrows = (int)min((int64_t)RT, a.n - r0); }
            int done = 0;
            while (done < nrows) {
                const int left = nrows - done;  // <= kTile = 64
                const int64_t base = __ldg(rp + r0 + done);
                // rp of rows done+1 .. done+left, two per lane, loaded together
                int64_t e0 = lane + 1 <= left ? __ldg(rp + r0 + done + lane + 1) - base : INT64_MAX;
                int64_t e1 = lane + 33 <= left ? __ldg(rp + r0 + done + lane + 33) - base : INT64_MAX;
                const unsigned m0 = __ballot_sync(0xffffffffu, e0 <= nnz_cap);
                const unsigned m1 = __ballot_sync(0xffffffffu, e1 <= nnz_cap);
                const int cnt = __popc(m0) + (m0 == 0xffffffffu ? __popc(m1) : 0);  // rp nondecreasing
                wait_stage();
                Ent *s_ent = reinterpret_cast<Ent *>(smem_raw + st * stage_bytes);
                int *s_rp = reinterpret_cast<int *>(smem_raw + st * stage_bytes + sizeof(Ent) * nnz_cap);
                if (cnt == 0) {  // one row longer than a stage
                    release(r0 + done, 1, 1);
                    done += 1;
                    continue;
                }
                if (lane == 0) s_rp[0] = 0;
                ARR_CHECK(cnt <= kTile);
                if (lane + 1 <= cnt) s_rp[lane + 1] = (int)e0;
                if (lane + 33 <= cnt) s_rp[lane + 33] = (int)e1;
                const int64_t nnz_t = __shfl_sync(0xffffffffu, cnt <= 32 ? e0 : e1, (cnt <= 32 ? cnt : cnt - 32) - 1);
                for (int64_t q0 = 0; q0 < nnz_t; q0 += 32 * UN) {
                    int32_t cv[UN];
                    double vv[UN];
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        const int64_t q = q0 + u * 32 + lane;
                        cv[u] = q < nnz_t ? __ldg(a.col + base + q) : 0;
                        vv[u] = q < nnz_t ? __ldg(a.val + base + q) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < UN; ++u) {
                        const int64_t q = q0 + u * 32 + lane;
                        if (q < nnz_t) {
                            ARR_CHECK(q < nnz_cap);
                            Ent e;
                            e.off = (int64_t)cv[u] * ld;
                            e.val = vv[u];
                            s_ent[q] = e;
                        }
                    }
                }
                release(r0 + done, cnt, 0);
                done += cnt;
            }
            if (DYN) {
                int64_t nx = 0;
                if (lane == 0) nx = (int64_t)gridDim.x + (int64_t)atomicAdd(a.sched, 1ull);
                t = __shfl_sync(0xffffffffu, nx, 0);
            } else {
                t += gridDim.x;
            }
        }
        wait_stage();
        release(-1, 0, 0);
        if (DYN && lane == 0) {
            __threadfence();
            if (atomicAdd(a.sched + 1, 1ull) == (unsigned long long)gridDim.x - 1) {
                a.sched[0] = 0;
                a.sched[1] = 0;
                __threadfence();
            }
        }
    } else {
        const int r = tid / TX;
        const int v0 = tid - r * TX;
        const bool active = r < R;
        double ss[NV][VEC];
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int e = 0; e < VEC; ++e) ss[v][e] = 0.0;
        const uint64_t pol_keep = policy_evict_last();
        const uint64_t pol_stream = policy_evict_first();
        int st = 0;
        for (;;) {
            nb_sync(1 + st, nall);
            const WsInfo info = s_info[st];
            if (info.r0 < 0) break;
            const Ent *s_ent = reinterpret_cast<const Ent *>(smem_raw + st * stage_bytes);
            const int *s_rp = reinterpret_cast<const int *>(smem_raw + st * stage_bytes + sizeof(Ent) * nnz_cap);
            if (info.mode == 0) {
                if (active)
                    tile_rows<VEC, NV, K, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>(a, info.r0, info.nrows, R, 0, r, TX, v0, wv,
                                                                            s_rp, s_ent, ss, pol_keep, pol_stream);
            } else if (active && r == 0) {
                // one row longer than a stage: CSR order straight from global memory
                using Vv = Vec<VEC>;
                using T = typename Vv::T;
                const int64_t i = info.r0;
                const int64_t p0 = __ldg(rp + i), p1 = __ldg(rp + i + 1);
                for (int v = 0; v < NV; ++v) {
                    const int vv = v0 + v * TX;
                    if (vv >= wv) continue;
                    T acc = Vv::zero();
                    for (int64_t p = p0; p < p1; ++p)
                        fma_vec<VEC>(acc, __ldg(a.val + p), Vv::ldg(a.Yin + (int64_t)__ldg(a.col + p) * ld + vv * VEC));
                    const T yi = Vv::ldg(a.Yin + i * ld + vv * VEC);
                    T yp = Vv::zero();
                    if (HAS_PREV) yp = Vv::ldcs(a.Yprev + i * a.ld_prev + vv * VEC);
                    T out;
                    for (int e = 0; e < VEC; ++e) {
                        const double sh = COLSHIFT ? __ldg(a.colshift + vv * VEC + e) : a.shift;
                        double o = epi(a.alpha, Vv::get(acc, e), sh, Vv::get(yi, e));
                        if (HAS_PREV)
                            o = fma(a.scale_mode == 2 ? a.beta * __ldg(a.colscale + vv * VEC + e) : a.beta,
                                    Vv::get(yp, e), o);
                        if (HAS_X) o = fma(a.gxa, a.Xa[i * a.ld_xa + vv * VEC + e], o);
                        if (a.scale_mode == 1) o *= __ldg(a.colscale + vv * VEC + e);
                        Vv::set(out, e, o);
                        if (SUMSQ) ss[v][e] = fma(o, o, ss[v][e]);
                    }
                    if (STORE) Vv::stcs(a.Yout + i * a.ld_out + vv * VEC, out);
                }
            }
            nb_arrive(3 + st, nall);
            st ^= 1;
        }
        if (SUMSQ) {
            // fixed-order reduction over the R row slots of each column (consumer threads only)
            double *red = reinterpret_cast<double *>(smem_raw);
            nb_sync(5, ncons);  // every consumer is past the last stage (the producer has exited the ring)
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (active) {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) red[(r * TX + v0) * VEC + e] = ss[v][e];
                }
                nb_sync(5, ncons);
                const int vv = v0 + v * TX;
                if (active && r == 0 && vv < wv) {
#pragma unroll
                    for (int e = 0; e < VEC; ++e) {
                        double sum = 0.0;
                        for (int q = 0; q < R; ++q) sum += red[(q * TX + v0) * VEC + e];
                        const int colid = vv * VEC + e;
                        if (colid < a.w) a.partials[(int64_t)blockIdx.x * a.w + colid] = sum;
                    }
                }
                nb_sync(5, ncons);
            }
        }
    }
}

template <int VEC, int NV, int K, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
int launch_t(arr_ctx *c, const SpmmArgs &a, int TX, int R, int wv) {
#if ARR_SPMM_WS
    // warp-specialised kernel where it measured faster on B200: >= 4 rows in flight per
    // CTA and single-chunk rows (cfg2: 116 -> 105 us); slower for R = 1 (cfg3, w = 550) and
    // for 27-point rows (cfg5), which keep spmm_tile_kernel
    if (R >= 4 && K <= 7) {
        auto kern = spmm_ws_kernel<VEC, NV, K, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>;
        const int ncons = ((R * TX + 31) / 32) * 32;
        const int RT = c->tile_rows;
        const size_t stage = ((sizeof(Ent) * (size_t)kWsCap + 4 * (size_t)(kTile + 2) + 15) & ~size_t(15));
        size_t smem = 2 * stage;
        const size_t red = 8 * (size_t)ncons * VEC;
        if (smem < red) smem = red;
        static LaunchCache cache;  // per instantiation (one device per process)
        const int occ = cached_occupancy(cache, kern, ncons + 32, smem);
        const int64_t ntiles = a.tile_row0 ? a.ntiles : (a.n + RT - 1) / RT;
        int64_t G = (int64_t)c->num_sms * occ;
        if (G > ntiles) G = ntiles;
        if (G < 1) G = 1;
        kern<<<(unsigned)G, ncons + 32, smem, c->stream>>>(a, TX, R, RT, wv, ntiles, kWsCap, ncons);
        c->launches++;
        c->last_kernel = "spmm_ws_kernel (CSR, warp-specialised)";
        return (int)G;
    }
#endif
    auto kern = spmm_tile_kernel<VEC, NV, K, HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>;
    const int nthr = ((R * TX + 31) / 32) * 32;
    const int RT = c->tile_rows;  // rows per tile in natural order (<= kTile)
    // smem: staged slice + relative row pointers; reused by the SUMSQ reduction
    size_t smem = ((sizeof(Ent) * (size_t)kNnzCap + 4 * (size_t)(kTile + 2) + 15) & ~size_t(15));
    const size_t red = 8 * (size_t)nthr * VEC;
    if (smem < red) smem = red;
    static LaunchCache cache;  // per instantiation (one device per process)
    const int occ = cached_occupancy(cache, kern, nthr, smem);
    const int64_t ntiles = a.tile_row0 ? a.ntiles : (a.n + RT - 1) / RT;
    int64_t G = (int64_t)c->num_sms * occ;
    if (G > ntiles) G = ntiles;
    if (G < 1) G = 1;
    kern<<<(unsigned)G, nthr, smem, c->stream>>>(a, TX, R, RT, wv, ntiles, kNnzCap);
    c->launches++;
    c->last_kernel = "spmm_tile_kernel (CSR)";
    return (int)G;
}

template <int VEC, int NV, int K>
int dispatch_flags(arr_ctx *c, const SpmmArgs &a, int TX, int R, int wv) {
    const bool prev = a.Yprev != nullptr, store = a.Yout != nullptr, ss = a.partials != nullptr,
               cs = a.colshift != nullptr, xa = a.Xa != nullptr;
    if (!xa) {
        if (prev && store && !ss && !cs) return launch_t<VEC, NV, K, true, true, false, false, false>(c, a, TX, R, wv);
        if (prev && store && ss && !cs) return launch_t<VEC, NV, K, true, true, true, false, false>(c, a, TX, R, wv);
        if (!prev && store && !ss && !cs) return launch_t<VEC, NV, K, false, true, false, false, false>(c, a, TX, R, wv);
        if (!prev && store && ss && !cs) return launch_t<VEC, NV, K, false, true, true, false, false>(c, a, TX, R, wv);
        if (!prev && !store && ss && cs) return launch_t<VEC, NV, K, false, false, true, true, false>(c, a, TX, R, wv);
    } else if (store && !cs) {  // the interpolant filter's Clenshaw steps (b_k = a_k X + 2 S b_{k+1} - b_{k+2})
        if (prev && !ss) return launch_t<VEC, NV, K, true, true, false, false, true>(c, a, TX, R, wv);
        if (prev && ss) return launch_t<VEC, NV, K, true, true, true, false, true>(c, a, TX, R, wv);
        if (!prev && !ss) return launch_t<VEC, NV, K, false, true, false, false, true>(c, a, TX, R, wv);
        if (!prev && ss) return launch_t<VEC, NV, K, false, true, true, false, true>(c, a, TX, R, wv);
    }
    return -1;
}

// Chunk size K from the longest row: whole rows in one chunk for the 3-, 5-
// and 7-point stencils, 3 chunks of 9 for the 27-point stencil, chunks of 8
// otherwise (irregular rows).
template <int VEC>
int dispatch_nv(arr_ctx *c, const SpmmArgs &a) {
    const int wv = (a.w + VEC - 1) / VEC;
    int TX = wv < kMaxThreads ? wv : kMaxThreads;
    if (c->col_split > 1 && wv / c->col_split >= 32) TX = (wv + c->col_split - 1) / c->col_split;  // NV > 1 per thread
    const int R = kMaxThreads / TX;
    const int nv = (wv + TX - 1) / TX;
    const int L = c->max_row_nnz;
    if (nv == 1) {
        if (L <= 3) return dispatch_flags<VEC, 1, 3>(c, a, TX, R, wv);
        if (L <= 5) return dispatch_flags<VEC, 1, 5>(c, a, TX, R, wv);
        if (L <= 7) return dispatch_flags<VEC, 1, 7>(c, a, TX, R, wv);
        if (L % 9 == 0) return dispatch_flags<VEC, 1, 9>(c, a, TX, R, wv);
        return dispatch_flags<VEC, 1, 8>(c, a, TX, R, wv);
    }
    if (nv == 2) return dispatch_flags<VEC, 2, 4>(c, a, TX, R, wv);
    if (nv <= 4) return dispatch_flags<VEC, 4, 2>(c, a, TX, R, wv);
    return -1;
}



__global__ void rowlen_max_kernel(const int64_t *__restrict__ rp, int64_t n, int *out) {
    int m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        { const int64_t L = rp[i + 1] - rp[i]; m = max(m, L > (1 << 30) ? (1 << 30) : (int)L); }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);  // integer max: order independent
}

__global__ void colnorm_finalize_kernel(const double *__restrict__ part, int nblk, int w,
                                        double *__restrict__ out, const double *__restrict__ mu_div) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= w) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * w + col];
    double r = sqrt(s);
    if (mu_div) r /= fmax(1.0, fabs(mu_div[col]));
    out[col] = r;
}

__global__ void colsum_kernel(const double *__restrict__ part, int nblk, int w, double *__restrict__ out) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= w) return;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += part[(int64_t)b * w + col];
    out[col] = s;
}

__global__ void colnorm_root_kernel(double *x, int w, const double *__restrict__ mu_div) {
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= w) return;
    double r = sqrt(x[col]);
    if (mu_div) r /= fmax(1.0, fabs(mu_div[col]));
    x[col] = r;
}

template <int VEC>
__global__ void scale_cols_kernel(const double *In, int64_t ld_in, double *Out, int64_t ld_out, int64_t n,
                                  int wv, const double *__restrict__ norms) {
    using V = Vec<VEC>;
    const int64_t total = n * wv;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / wv;
        const int vv = (int)(t - i * wv);
        typename V::T x = V::ldcs(In + i * ld_in + vv * VEC);
#pragma unroll
        for (int e = 0; e < VEC; ++e) V::set(x, e, V::get(x, e) / norms[vv * VEC + e]);
        V::stcs(Out + i * ld_out + vv * VEC, x);
    }
}

__global__ void gershgorin_kernel(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                  const double *__restrict__ val, int64_t n, double sign, double *__restrict__ part) {
    // min_i (sign*A_ii - sum_{j != i} |A_ij|): the Gershgorin lower bound of sign*A
    double m = INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double dg = 0.0, off = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (col[p] == i) dg += val[p];
            else off += fabs(val[p]);
        }
        m = fmin(m, sign * dg - off);
    }
    __shared__ double red[256];
    red[threadIdx.x] = m;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] = fmin(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void min_finalize_kernel(const double *part, int nblk, double *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double m = INFINITY;
        for (int b = 0; b < nblk; ++b) m = fmin(m, part[b]);
        *out = m;
    }
}

__global__ void check_norms_kernel(const double *norms, int w, int *bad) {
    int flag = 0;
    for (int cidx = threadIdx.x; cidx < w; cidx += blockDim.x) {
        const double x = norms[cidx];
        if (!(x > 0.0) || !isfinite(x)) flag = 1;
    }
    flag = __syncthreads_or(flag);
    if (threadIdx.x == 0) *bad = flag;
}

__global__ void copy_rows_kernel(const double *__restrict__ src, int64_t lds, double *__restrict__ dst,
                                 int64_t ldd, int64_t n, int w) {
    const int64_t total = n * (int64_t)w;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / w;
        const int cc = (int)(t - i * w);
        dst[i * ldd + cc] = src[i * lds + cc];
    }
}

bool vec2_ok(const void *p, int64_t ld) { return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0); }
bool vec4_ok(const void *p, int64_t ld) { return ((uintptr_t)p % 32 == 0) && (ld % 4 == 0); }

}  // namespace

void launch_rowlen_max(arr_ctx *c, int *dev_out) {
    cudaMemsetAsync(dev_out, 0, sizeof(int), c->stream);
    int64_t blocks = (c->A.n + 255) / 256;
    if (blocks > (int64_t)c->num_sms * 4) blocks = (int64_t)c->num_sms * 4;
    if (blocks < 1) blocks = 1;
    rowlen_max_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(c->A.row_ptr, c->A.n, dev_out);
    c->launches++;
}

int launch_spmm(arr_ctx *c, const SpmmArgs &a_in) {
    SpmmArgs a = a_in;
    a.nnz = c->A.nnz;
    a.sched = c->sched;
    if (!a.tile_row0 && c->tile_row0 && a.n == c->A.n) {
        a.tile_row0 = c->tile_row0;
        a.tile_len = c->tile_len;
        a.ntiles = c->ntiles;
    }
    bool v2 = (a.w % 2 == 0) && vec2_ok(a.Yin, a.ld_in);
    if (a.Yprev) v2 = v2 && vec2_ok(a.Yprev, a.ld_prev);
    if (a.Yout) v2 = v2 && vec2_ok(a.Yout, a.ld_out);
    if (a.Xa) v2 = v2 && vec2_ok(a.Xa, a.ld_xa);
    c->spmm_blocks++;
    if (c->st.on && !a.tile_row0) {  // declared stencil operator (eig_set_stencil): the 2.5-D blocked path
        const int g = launch_spmm_stencil(c, a);
        if (g >= 0) return g;
    }
#if ARR_SPMM_V4
    bool v4 = (a.w % 4 == 0) && vec4_ok(a.Yin, a.ld_in);
    if (a.Yprev) v4 = v4 && vec4_ok(a.Yprev, a.ld_prev);
    if (a.Yout) v4 = v4 && vec4_ok(a.Yout, a.ld_out);
    if (a.Xa) v4 = v4 && vec4_ok(a.Xa, a.ld_xa);
    if (v4) return dispatch_nv<4>(c, a);
#endif
    return v2 ? dispatch_nv<2>(c, a) : dispatch_nv<1>(c, a);
}

void launch_colnorm_finalize(arr_ctx *c, const double *partials, int nblk, int32_t w, double *out,
                             const double *mu_div) {
    colnorm_finalize_kernel<<<(w + 127) / 128, 128, 0, c->stream>>>(partials, nblk, w, out, mu_div);
    c->launches++;
}

void launch_colsum(arr_ctx *c, const double *partials, int nblk, int32_t w, double *out) {
    colsum_kernel<<<(w + 127) / 128, 128, 0, c->stream>>>(partials, nblk, w, out);
    c->launches++;
}

void launch_colnorm_root(arr_ctx *c, double *x, int32_t w, const double *mu_div) {
    colnorm_root_kernel<<<(w + 127) / 128, 128, 0, c->stream>>>(x, w, mu_div);
    c->launches++;
}

namespace {
__global__ void recip_kernel(const double *__restrict__ x, int w, double *__restrict__ out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < w) out[i] = 1.0 / x[i];
}
}  // namespace

void launch_recip(arr_ctx *c, const double *x, int32_t w, double *out) {
    recip_kernel<<<(w + 255) / 256, 256, 0, c->stream>>>(x, w, out);
    c->launches++;
}

void launch_scale_cols(arr_ctx *c, const double *In, int64_t ld_in, double *Out, int64_t ld_out, int64_t n,
                       int32_t w, const double *norms) {
    const bool v2 = (w % 2 == 0) && vec2_ok(In, ld_in) && vec2_ok(Out, ld_out);
    const int wv = v2 ? w / 2 : w;
    int64_t blocks = (n * wv + 255) / 256;
    const int64_t cap = (int64_t)c->num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (v2)
        scale_cols_kernel<2><<<(unsigned)blocks, 256, 0, c->stream>>>(In, ld_in, Out, ld_out, n, wv, norms);
    else
        scale_cols_kernel<1><<<(unsigned)blocks, 256, 0, c->stream>>>(In, ld_in, Out, ld_out, n, wv, norms);
    c->launches++;
}

void launch_gershgorin(arr_ctx *c, double *partial, int *nblk_out) {
    int64_t blocks = (c->A.n + 255) / 256;
    const int64_t cap = (int64_t)c->num_sms * 4;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    gershgorin_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(c->A.row_ptr, c->A.col_idx, c->A.val, c->A.n,
                                                              (double)c->sign, partial);
    c->launches++;
    *nblk_out = (int)blocks;
}

void launch_min_finalize(arr_ctx *c, const double *partial, int nblk, double *out) {
    min_finalize_kernel<<<1, 32, 0, c->stream>>>(partial, nblk, out);
    c->launches++;
}

void launch_check_norms(arr_ctx *c, const double *norms, int32_t w, int *bad) {
    check_norms_kernel<<<1, 256, 0, c->stream>>>(norms, w, bad);
    c->launches++;
}

void launch_copy_rows(arr_ctx *c, const double *src, int64_t lds, double *dst, int64_t ldd, int64_t n,
                      int32_t w) {
    int64_t blocks = (n * (int64_t)w + 255) / 256;
    const int64_t cap = (int64_t)c->num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    copy_rows_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(src, lds, dst, ldd, n, w);
    c->launches++;
}

// ---------------------------------------------------------------- schedule check
namespace {
__global__ void sched_mark_kernel(const int64_t *row0, const int32_t *len, int64_t ntiles, int64_t n, int *marks,
                                  int *bad) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < ntiles;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = row0[t];
        const int l = len[t];
        if (l < 1 || l > kTile || r < 0 || r + l > n) {
            atomicOr(bad, 1);
            continue;
        }
        for (int q = 0; q < l; ++q) atomicAdd(marks + r + q, 1);
    }
}
__global__ void sched_verify_kernel(const int *marks, int64_t n, int *bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (marks[i] != 1) atomicOr(bad, 1);
}
}  // namespace

void launch_schedule_check(arr_ctx *c, const int64_t *row0, const int32_t *len, int64_t ntiles, int *marks,
                           int *bad) {
    cudaMemsetAsync(marks, 0, sizeof(int) * (size_t)c->A.n, c->stream);
    cudaMemsetAsync(bad, 0, sizeof(int), c->stream);
    const unsigned g = (unsigned)c->num_sms * 4;
    sched_mark_kernel<<<g, 256, 0, c->stream>>>(row0, len, ntiles, c->A.n, marks, bad);
    sched_verify_kernel<<<g, 256, 0, c->stream>>>(marks, c->A.n, bad);
    c->launches += 2;
}
