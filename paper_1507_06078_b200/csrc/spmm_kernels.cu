// Fused CSR x row-major-block kernels for sm_100a: the Chebyshev filter degree
// (Eq. cheby-poly P:377-383 on the map of Eq. rhod, Alg. Arrabit2
// line P:1486), the augmentation SpMM (Alg. ARR) and the residual pass
// (Eq. resi).  HBM-bound: every degree reads A once,
// gathers Y_j rows through L1/L2, streams Y_{j-1} in and Y_{j+1} out with
// evict-first hints, and optionally emits deterministic column sums of squares.
#include <math.h>

#include "internal.cuh"

namespace {

constexpr int kThreads = 256;

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
    using T = double;
    static __device__ __forceinline__ T zero() { return 0.0; }
    static __device__ __forceinline__ T ldg(const double *p) { return __ldg(p); }
    static __device__ __forceinline__ T ldcs(const double *p) { return __ldcs(p); }
    static __device__ __forceinline__ void stcs(double *p, T v) { __stcs(p, v); }
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
    static __device__ __forceinline__ double get(const T &v, int e) { return e ? v.y : v.x; }
    static __device__ __forceinline__ void set(T &v, int e, double x) {
        if (e) v.y = x; else v.x = x;
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

// Thread (r, v0) of a CTA owns row r of each row group and the vector columns
// v0, v0+TX, ... (NV of them).  Row groups of R rows are visited grid-stride so
// the rows active on the chip at any time form one contiguous window (L2 reuse
// of gathered neighbour rows).  Per-row sums run in CSR order (fixed, partition
// independent).
template <int VEC, int NV, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT>
__global__ void __launch_bounds__(kThreads) spmm_fused_kernel(SpmmArgs a, int TX, int R, int wv,
                                                               int64_t ngroups) {
    using V = Vec<VEC>;
    using T = typename V::T;
    const int tid = threadIdx.x;
    const int r = tid / TX;
    const int v0 = tid - r * TX;
    const bool active = r < R;
    double ss[NV][VEC];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
        for (int e = 0; e < VEC; ++e) ss[v][e] = 0.0;

    if (active) {
        const int64_t *__restrict__ rp = a.row_ptr;
        const int32_t *__restrict__ col = a.col;
        const double *__restrict__ val = a.val;
        const double *__restrict__ Yin = a.Yin;
        for (int64_t g = blockIdx.x; g < ngroups; g += gridDim.x) {
            const int64_t i = g * R + r;
            if (i >= a.n) break;
            const int64_t p0 = rp[i];
            const int64_t p1 = rp[i + 1];
            T acc[NV];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = V::zero();
            int64_t p = p0;
            constexpr int U = (NV == 1) ? 4 : 2;
            for (; p + U <= p1; p += U) {
                int jj[U];
                double aa[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    jj[u] = __ldg(col + p + u);
                    aa[u] = __ldg(val + p + u);
                }
                T x[U][NV];
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int v = 0; v < NV; ++v) {
                        const int vv = v0 + v * TX;
                        x[u][v] = (vv < wv) ? V::ldg(Yin + (int64_t)jj[u] * a.ld_in + vv * VEC) : V::zero();
                    }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int v = 0; v < NV; ++v) fma_vec<VEC>(acc[v], aa[u], x[u][v]);
            }
            for (; p < p1; ++p) {
                const int j = __ldg(col + p);
                const double av = __ldg(val + p);
#pragma unroll
                for (int v = 0; v < NV; ++v) {
                    const int vv = v0 + v * TX;
                    if (vv < wv) fma_vec<VEC>(acc[v], av, V::ldg(Yin + (int64_t)j * a.ld_in + vv * VEC));
                }
            }
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const int vv = v0 + v * TX;
                if (vv >= wv) continue;
                const T yi = V::ldg(Yin + i * a.ld_in + vv * VEC);
                T yp = V::zero();
                if (HAS_PREV) yp = V::ldcs(a.Yprev + i * a.ld_prev + vv * VEC);
                T out;
#pragma unroll
                for (int e = 0; e < VEC; ++e) {
                    const double sh = COLSHIFT ? __ldg(a.colshift + vv * VEC + e) : a.shift;
                    double o = a.alpha * (V::get(acc[v], e) - sh * V::get(yi, e));
                    if (HAS_PREV) o += a.beta * V::get(yp, e);
                    V::set(out, e, o);
                    if (SUMSQ) ss[v][e] = fma(o, o, ss[v][e]);
                }
                if (STORE) V::stcs(a.Yout + i * a.ld_out + vv * VEC, out);
            }
        }
    }
    if (SUMSQ) {
        // fixed-order block reduction over the R row-threads of each column
        __shared__ double red[kThreads * VEC];
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
                    double s = 0.0;
                    for (int rr = 0; rr < R; ++rr) s += red[(rr * TX + v0) * VEC + e];
                    const int colid = vv * VEC + e;
                    if (colid < a.w) a.partials[(int64_t)blockIdx.x * a.w + colid] = s;
                }
            }
        }
    }
}

template <int VEC, int NV, bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT>
int launch_t(arr_ctx *c, const SpmmArgs &a, int TX, int R, int wv) {
    auto kern = spmm_fused_kernel<VEC, NV, HAS_PREV, STORE, SUMSQ, COLSHIFT>;
    static int occ = -1;  // per instantiation
    if (occ < 0) {
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, kThreads, 0);
        occ = o > 0 ? o : 1;
    }
    const int64_t ngroups = (a.n + R - 1) / R;
    int64_t G = (int64_t)c->num_sms * occ;
    if (G > ngroups) G = ngroups;
    if (G < 1) G = 1;
    kern<<<(unsigned)G, kThreads, 0, c->stream>>>(a, TX, R, wv, ngroups);
    c->launches++;
    return (int)G;
}

template <int VEC, int NV>
int dispatch_flags(arr_ctx *c, const SpmmArgs &a, int TX, int R, int wv) {
    const bool prev = a.Yprev != nullptr, store = a.Yout != nullptr, ss = a.partials != nullptr,
               cs = a.colshift != nullptr;
    if (prev && store && !ss && !cs) return launch_t<VEC, NV, true, true, false, false>(c, a, TX, R, wv);
    if (prev && store && ss && !cs) return launch_t<VEC, NV, true, true, true, false>(c, a, TX, R, wv);
    if (!prev && store && !ss && !cs) return launch_t<VEC, NV, false, true, false, false>(c, a, TX, R, wv);
    if (!prev && store && ss && !cs) return launch_t<VEC, NV, false, true, true, false>(c, a, TX, R, wv);
    if (!prev && !store && ss && cs) return launch_t<VEC, NV, false, false, true, true>(c, a, TX, R, wv);
    return -1;
}

template <int VEC>
int dispatch_nv(arr_ctx *c, const SpmmArgs &a) {
    const int wv = (a.w + VEC - 1) / VEC;
    const int TX = wv < kThreads ? wv : kThreads;
    const int R = kThreads / TX;
    const int nv = (wv + TX - 1) / TX;
    if (nv == 1) return dispatch_flags<VEC, 1>(c, a, TX, R, wv);
    if (nv == 2) return dispatch_flags<VEC, 2>(c, a, TX, R, wv);
    if (nv <= 4) return dispatch_flags<VEC, 4>(c, a, TX, R, wv);
    return -1;
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
                                  const double *__restrict__ val, int64_t n, double *__restrict__ part) {
    double m = INFINITY;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double dg = 0.0, off = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            if (col[p] == i) dg += val[p];
            else off += fabs(val[p]);
        }
        m = fmin(m, dg - off);
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

}  // namespace

int launch_spmm(arr_ctx *c, const SpmmArgs &a) {
    bool v2 = (a.w % 2 == 0) && vec2_ok(a.Yin, a.ld_in);
    if (a.Yprev) v2 = v2 && vec2_ok(a.Yprev, a.ld_prev);
    if (a.Yout) v2 = v2 && vec2_ok(a.Yout, a.ld_out);
    c->spmm_blocks++;
    return v2 ? dispatch_nv<2>(c, a) : dispatch_nv<1>(c, a);
}

void launch_colnorm_finalize(arr_ctx *c, const double *partials, int nblk, int32_t w, double *out,
                             const double *mu_div) {
    colnorm_finalize_kernel<<<(w + 127) / 128, 128, 0, c->stream>>>(partials, nblk, w, out, mu_div);
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
                                                              partial);
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
