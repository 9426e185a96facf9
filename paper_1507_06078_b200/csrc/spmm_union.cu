// Union-staged fused SpMM (the filter degree / augmentation / residual SpMM of
// spmm_kernels.cu, Eq. cheby-poly, with the same per-row CSR-order
// arithmetic) for matrices whose neighbouring rows share columns (stencils,
// banded and mesh matrices).
//
// The tiled kernels gather Y_j[col, :] once per non-zero through L1/L2: a 27-point
// row reads 27 X rows although a tile of consecutive grid points needs each
// neighbour row only once.  Here a tile is a contiguous range of rows whose
// non-zeros reference U distinct columns; U is precomputed once per tile
// (union_prep_kernel: sort + unique of the tile's column indices, and a 16-bit
// local index per non-zero).  Per column panel of PW doubles the CTA stages the U
// rows Y_j[u, panel] into shared memory with cp.async (each distinct row read once)
// and computes every row of the tile from shared memory.  The tile's CSR values and
// local indices are staged once and reused by every panel.  Per-row sums run over
// the row's non-zeros in CSR order with the same fma sequence as the tiled kernels,
// so the results are bitwise identical to theirs.
//
// Status: opt-in (ARRABIT_UNION=1).  Measured on B200 (profiles/r01_experiments/union.log):
// cfg2 182 us vs 103 us per degree, cfg3 6.8 ms vs 3.7 ms, cfg5 121 ms vs 79 ms -- the
// per-panel staging barriers and narrow (64-128 B) panel rows cost more than the saved
// L1/L2 gather traffic; kept, parity-tested, as the starting point of a pipelined
// (producer-warp / TMA) variant.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.cuh"

namespace {

constexpr int kUThreads = 256;
constexpr int kUCap = 4096;  // non-zeros per union tile (16-bit local indices, bitonic sort size)

__device__ __forceinline__ void ca16u(void *smem, const void *gmem, int bytes) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}

// One CTA per tile: sorted distinct columns of the tile -> ucol[base ..), local
// index of every non-zero -> loc[base + p], count -> ucnt[t] (-1: tile too large).
__global__ void __launch_bounds__(512) union_prep_kernel(const int64_t *__restrict__ rp,
                                                               const int32_t *__restrict__ col,
                                                               const int64_t *__restrict__ t_r0,
                                                               const int32_t *__restrict__ t_len, int32_t *ucol,
                                                               uint16_t *loc, int32_t *ucnt) {
    constexpr int kPT = 512;  // prep threads
    __shared__ int keys[kUCap];
    __shared__ int scan[kPT + 1];
    const int t = blockIdx.x, tid = threadIdx.x;
    const int64_t r0 = t_r0[t];
    const int64_t base = rp[r0], nz = rp[r0 + t_len[t]] - base;
    if (nz > kUCap || nz < 1) {
        if (tid == 0) ucnt[t] = nz < 1 ? 0 : -1;
        return;
    }
    int P2 = 1;
    while (P2 < nz) P2 <<= 1;
    for (int i = tid; i < P2; i += kPT) keys[i] = i < nz ? col[base + i] : 0x7fffffff;
    __syncthreads();
    // bitonic sort (ascending)
    for (int k = 2; k <= P2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = tid; i < P2; i += kPT) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const int a = keys[i], b = keys[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { keys[i] = b; keys[ixj] = a; }
                }
            }
            __syncthreads();
        }
    // distinct values: flag, block-wide exclusive scan (each thread owns a contiguous chunk)
    const int per = (P2 + kPT - 1) / kPT;
    const int i0 = tid * per, i1 = min(P2, i0 + per);
    int cnt = 0;
    for (int i = i0; i < i1; ++i)
        if (i < nz && (i == 0 || keys[i] != keys[i - 1])) ++cnt;
    scan[tid + 1] = cnt;
    if (tid == 0) scan[0] = 0;
    __syncthreads();
    if (tid == 0)
        for (int q = 1; q <= kPT; ++q) scan[q] += scan[q - 1];
    __syncthreads();
    const int U = scan[kPT];
    int o = scan[tid];
    int vals[8];  // per <= kUCap / kPT = 8
    int nv = 0;
    for (int i = i0; i < i1; ++i)
        if (i < nz && (i == 0 || keys[i] != keys[i - 1])) vals[nv++] = keys[i];
    __syncthreads();  // every thread has read its keys; compact in place
    for (int q = 0; q < nv; ++q) keys[o + q] = vals[q];
    __syncthreads();
    for (int u = tid; u < U; u += kPT) ucol[base + u] = keys[u];
    for (int p = tid; p < nz; p += kPT) {
        const int cv = col[base + p];
        int lo = 0, hi = U - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (keys[mid] < cv) lo = mid + 1; else hi = mid;
        }
        loc[base + p] = (uint16_t)lo;
    }
    if (tid == 0) ucnt[t] = U;
}

template <bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
__global__ void __launch_bounds__(kUThreads, 4) spmm_union_kernel(SpmmArgs a, UnionPlan u, int PW) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *s_x = reinterpret_cast<double *>(smem_raw);                        // [2][umax][PW] (panel ring)
    double *s_val = s_x + 2 * (size_t)u.umax * PW;                               // [nzmax]
    double *s_red = s_val + u.nzmax;                                             // [kUThreads/32][PW]
    int *s_rp = reinterpret_cast<int *>(s_red + (kUThreads / 32) * PW);          // [rtmax + 1]
    int *s_uc = s_rp + u.rtmax + 1;                                              // [umax]
    uint16_t *s_loc = reinterpret_cast<uint16_t *>(s_uc + u.umax);              // [nzmax]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int PV = PW / 2;  // 16-byte vectors per panel row
    const int64_t ld = a.ld_in;
    if (SUMSQ)
        for (int cidx = tid; cidx < a.w; cidx += kUThreads) a.partials[(int64_t)blockIdx.x * a.w + cidx] = 0.0;
    for (int64_t t = blockIdx.x; t < u.ntiles; t += gridDim.x) {
        const int64_t r0 = u.r0[t];
        const int len = u.len[t];
        const int U = u.cnt[t];
        const int64_t base = __ldg(a.row_ptr + r0);
        __syncthreads();  // previous tile done with the staged CSR
        for (int q = tid; q <= len; q += kUThreads) s_rp[q] = (int)(__ldg(a.row_ptr + r0 + q) - base);
        for (int q = tid; q < U; q += kUThreads) s_uc[q] = u.ucol[base + q];
        __syncthreads();
        const int nz = s_rp[len];
        for (int q = tid; q < nz; q += kUThreads) {
            s_val[q] = __ldg(a.val + base + q);
            s_loc[q] = u.loc[base + q];
        }
        // column panels through a two-buffer cp.async ring: panel q+1 is in flight
        // while panel q is computed
        const int npan = (a.w + PW - 1) / PW;
        auto stage = [&](int q) {
            const int c0 = q * PW;
            const int nvec = min(PV, (a.w - c0) >> 1);
            double *dst = s_x + (size_t)(q & 1) * u.umax * PW;
            for (int idx = tid; idx < U * PV; idx += kUThreads) {
                const int uu = idx / PV, ch = idx - uu * PV;
                const bool ok = ch < nvec;
                const double *src = ok ? a.Yin + (int64_t)s_uc[uu] * ld + c0 + 2 * ch : a.Yin;
                ca16u(dst + (size_t)uu * PW + 2 * ch, src, ok ? 16 : 0);
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        stage(0);
        for (int q = 0; q < npan; ++q) {
            const int c0 = q * PW;
            const int nvec = min(PV, (a.w - c0) >> 1);
            if (q + 1 < npan) {
                stage(q + 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            __syncthreads();
            const double *xb = s_x + (size_t)(q & 1) * u.umax * PW;
            double ss0 = 0.0, ss1 = 0.0;
            const int v = tid % PV;  // kUThreads is a multiple of PV: fixed column pair per thread
            for (int slot = tid; slot < len * PV; slot += kUThreads) {
                const int r = slot / PV;
                if (v >= nvec) continue;
                const int colv = c0 + 2 * v;
                double2 acc = make_double2(0.0, 0.0);
                for (int p = s_rp[r]; p < s_rp[r + 1]; ++p) {
                    const double av = s_val[p];
                    const double2 x = *reinterpret_cast<const double2 *>(xb + (size_t)s_loc[p] * PW + 2 * v);
                    acc.x = fma(av, x.x, acc.x);
                    acc.y = fma(av, x.y, acc.y);
                }
                const int64_t i = r0 + r;
                const double2 yi = __ldg(reinterpret_cast<const double2 *>(a.Yin + i * ld + colv));
                const double sh0 = COLSHIFT ? __ldg(a.colshift + colv) : a.shift;
                const double sh1 = COLSHIFT ? __ldg(a.colshift + colv + 1) : a.shift;
                double o0 = a.alpha * (acc.x - sh0 * yi.x);
                double o1 = a.alpha * (acc.y - sh1 * yi.y);
                if (HAS_PREV) {
                    const double2 yp = __ldcs(reinterpret_cast<const double2 *>(a.Yprev + i * a.ld_prev + colv));
                    o0 += a.beta * yp.x;
                    o1 += a.beta * yp.y;
                }
                if (HAS_X) {
                    o0 += a.gxa * a.Xa[i * a.ld_xa + colv];
                    o1 += a.gxa * a.Xa[i * a.ld_xa + colv + 1];
                }
                if (STORE) __stcs(reinterpret_cast<double2 *>(a.Yout + i * a.ld_out + colv), make_double2(o0, o1));
                if (SUMSQ) { ss0 = fma(o0, o0, ss0); ss1 = fma(o1, o1, ss1); }
            }
            if (SUMSQ) {
                // fixed-order reduction: lanes with the same v inside the warp, then warps
                for (int off = PV; off < 32; off <<= 1) {
                    ss0 += __shfl_down_sync(0xffffffffu, ss0, off);
                    ss1 += __shfl_down_sync(0xffffffffu, ss1, off);
                }
                if (lane < PV) {
                    s_red[warp * PW + 2 * lane] = ss0;
                    s_red[warp * PW + 2 * lane + 1] = ss1;
                }
                __syncthreads();
                if (tid < 2 * nvec) {
                    double s = 0.0;
                    for (int qq = 0; qq < kUThreads / 32; ++qq) s += s_red[qq * PW + tid];
                    a.partials[(int64_t)blockIdx.x * a.w + c0 + tid] += s;
                }
            }
            __syncthreads();  // panel q's buffer (and s_red) free for panel q+2
        }
    }
}

}  // namespace

size_t union_smem_bytes(int umax, int rtmax, int nzmax, int PW) {
    return sizeof(double) * (2 * (size_t)umax * PW + nzmax + (kUThreads / 32) * PW) + sizeof(int) * (rtmax + 1 + umax) +
           sizeof(uint16_t) * (size_t)nzmax + 16;
}

// Build the union plan for the ctx's current tiling (natural order, or the schedule's
// tiles merged into contiguous runs of up to ARRABIT_UNION_ROWS rows).  Returns false
// (plan off) when the matrix has too little column sharing or a tile does not fit.
bool union_prepare(arr_ctx *c) {
    UnionPlan &u = c->uplan;
    union_release(c);
    // opt-in (ARRABIT_UNION=1): measured slower than the tiled kernels on B200
    const char *env = getenv("ARRABIT_UNION");
    if (!env || env[0] != '1') return false;
    if (c->nranks > 1 || c->A.n < 1 || c->A.nnz < 1) return false;
    const int64_t n = c->A.n;
    int rows_max = 64;
    if (const char *e = getenv("ARRABIT_UNION_ROWS")) rows_max = std::max(1, std::min(1024, atoi(e)));
    std::vector<int64_t> rp(n + 1);
    if (cudaMemcpy(rp.data(), c->A.row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
        return false;
    // candidate runs: the schedule's tiles in order (contiguous successors merged) or natural order
    std::vector<int64_t> s0;
    std::vector<int32_t> sl;
    if (c->tile_row0) {
        s0.resize(c->ntiles);
        sl.resize(c->ntiles);
        if (cudaMemcpy(s0.data(), c->tile_row0, sizeof(int64_t) * c->ntiles, cudaMemcpyDeviceToHost) != cudaSuccess ||
            cudaMemcpy(sl.data(), c->tile_len, sizeof(int32_t) * c->ntiles, cudaMemcpyDeviceToHost) != cudaSuccess)
            return false;
    } else {
        s0.push_back(0);
        sl.push_back((int32_t)std::min<int64_t>(n, INT32_MAX));
    }
    std::vector<int64_t> t0;
    std::vector<int32_t> tl;
    for (size_t q = 0; q < s0.size(); ++q) {
        int64_t r = s0[q], end = s0[q] + sl[q];
        // extend the run with contiguous successors
        while (q + 1 < s0.size() && s0[q + 1] == end) end += sl[++q];
        while (r < end) {
            int64_t e = r + 1;
            if (rp[e] - rp[r] > kUCap) return false;  // one row longer than a tile
            while (e < end && e - r < rows_max && rp[e + 1] - rp[r] <= kUCap) ++e;
            t0.push_back(r);
            tl.push_back((int32_t)(e - r));
            r = e;
        }
    }
    u.ntiles = (int64_t)t0.size();
    const size_t nnz = (size_t)c->A.nnz;
    int rtmax = 0, nzmax = 0;
    for (size_t q = 0; q < t0.size(); ++q) {
        rtmax = std::max(rtmax, (int)tl[q]);
        nzmax = std::max(nzmax, (int)(rp[t0[q] + tl[q]] - rp[t0[q]]));
    }
    if (cudaMallocAsync((void **)&u.r0, sizeof(int64_t) * u.ntiles, c->stream) != cudaSuccess ||
        cudaMallocAsync((void **)&u.len, sizeof(int32_t) * u.ntiles, c->stream) != cudaSuccess ||
        cudaMallocAsync((void **)&u.cnt, sizeof(int32_t) * u.ntiles, c->stream) != cudaSuccess ||
        cudaMallocAsync((void **)&u.ucol, sizeof(int32_t) * nnz, c->stream) != cudaSuccess ||
        cudaMallocAsync((void **)&u.loc, sizeof(uint16_t) * nnz, c->stream) != cudaSuccess) {
        union_release(c);
        return false;
    }
    cudaMemcpyAsync(u.r0, t0.data(), sizeof(int64_t) * u.ntiles, cudaMemcpyHostToDevice, c->stream);
    cudaMemcpyAsync(u.len, tl.data(), sizeof(int32_t) * u.ntiles, cudaMemcpyHostToDevice, c->stream);
    union_prep_kernel<<<(unsigned)u.ntiles, 512, 0, c->stream>>>(c->A.row_ptr, c->A.col_idx, u.r0, u.len,
                                                                       u.ucol, u.loc, u.cnt);
    c->launches++;
    std::vector<int32_t> cnt(u.ntiles);
    if (cudaMemcpyAsync(cnt.data(), u.cnt, sizeof(int32_t) * u.ntiles, cudaMemcpyDeviceToHost, c->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
        union_release(c);
        return false;
    }
    int64_t usum = 0;
    int umax = 0;
    for (int32_t x : cnt) {
        if (x < 0) { union_release(c); return false; }
        usum += x;
        umax = std::max(umax, (int)x);
    }
    double min_ratio = 1.3;
    if (const char *e = getenv("ARRABIT_UNION_MIN")) min_ratio = atof(e);
    const double ratio = usum > 0 ? (double)nnz / (double)usum : 0.0;
    // panel width: the widest of 32/16/8 doubles whose two staging buffers fit four CTAs
    // per SM, else two
    int PW = 0;
    for (size_t lim : {(size_t)54 * 1024, (size_t)110 * 1024}) {
        for (int pw : {32, 16, 8})
            if (union_smem_bytes(umax, rtmax, nzmax, pw) <= lim) { PW = pw; break; }
        if (PW) break;
    }
    if (const char *e = getenv("ARRABIT_UNION_PW")) {
        const int pw = atoi(e);
        if ((pw == 8 || pw == 16 || pw == 32) && union_smem_bytes(umax, rtmax, nzmax, pw) <= 220 * 1024) PW = pw;
    }
    if (getenv("ARRABIT_UNION_VERBOSE"))
        fprintf(stderr, "[union] tiles %lld rows<=%d nnz<=%d U<=%d reuse %.3f PW %d smem %zu -> %s\n",
                (long long)u.ntiles, rtmax, nzmax, umax, ratio, PW, PW ? union_smem_bytes(umax, rtmax, nzmax, PW) : 0,
                (PW == 0 || ratio < min_ratio || umax > 65535) ? "off" : "on");
    if (PW == 0 || ratio < min_ratio || umax > 65535) {
        union_release(c);
        return false;
    }
    u.umax = umax;
    u.rtmax = rtmax;
    u.nzmax = nzmax;
    u.pw = PW;
    u.ratio = ratio;
    u.on = true;
    return true;
}

void union_release(arr_ctx *c) {
    UnionPlan &u = c->uplan;
    void *ptrs[] = {u.r0, u.len, u.cnt, u.ucol, u.loc};
    for (void *p : ptrs)
        if (p) cudaFreeAsync(p, c->stream);
    u = UnionPlan{};
}

template <bool HAS_PREV, bool STORE, bool SUMSQ, bool COLSHIFT, bool HAS_X>
static int launch_union_t(arr_ctx *c, const SpmmArgs &a) {
    const UnionPlan &u = c->uplan;
    const size_t smem = union_smem_bytes(u.umax, u.rtmax, u.nzmax, u.pw);
    auto kern = spmm_union_kernel<HAS_PREV, STORE, SUMSQ, COLSHIFT, HAS_X>;
    static LaunchCache cache;
    const int per_sm = cached_occupancy(cache, kern, kUThreads, smem);
    int64_t grid = (int64_t)c->num_sms * per_sm;
    if (grid > u.ntiles) grid = u.ntiles;
    if (grid < 1) grid = 1;
    kern<<<(unsigned)grid, kUThreads, smem, c->stream>>>(a, u, u.pw);
    c->launches++;
    return (int)grid;
}

// Returns the grid size, or -1 when the union path does not apply to this launch.
int launch_spmm_union(arr_ctx *c, const SpmmArgs &a) {
    if (!c->uplan.on || a.n != c->A.n || a.row_ptr != c->A.row_ptr || (a.w & 1)) return -1;
    auto al = [](const void *p, int64_t ld) { return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0); };
    if (!al(a.Yin, a.ld_in) || (a.Yprev && !al(a.Yprev, a.ld_prev)) || (a.Yout && !al(a.Yout, a.ld_out)) ||
        (a.Xa && !al(a.Xa, a.ld_xa)))
        return -1;
    const bool hp = a.Yprev != nullptr, st = a.Yout != nullptr, sq = a.partials != nullptr,
               cs = a.colshift != nullptr, hx = a.Xa != nullptr;
    if (hx) return hp && st && !sq && !cs ? launch_union_t<true, true, false, false, true>(c, a)
                                          : (hp && st && sq && !cs ? launch_union_t<true, true, true, false, true>(c, a)
                                                                   : -1);
    if (cs) return (!hp && !st && sq) ? launch_union_t<false, false, true, true, false>(c, a) : -1;
    if (hp) return st ? (sq ? launch_union_t<true, true, true, false, false>(c, a)
                            : launch_union_t<true, true, false, false, false>(c, a))
                      : -1;
    if (st) return sq ? launch_union_t<false, true, true, false, false>(c, a)
                      : launch_union_t<false, true, false, false, false>(c, a);
    return sq ? launch_union_t<false, false, true, false, false>(c, a) : -1;
}
