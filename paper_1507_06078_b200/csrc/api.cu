// C-ABI of libarrabit (include/arrabit.h): context, workspace, and the
// composition of the kernels into filter_step / orthonormalize / arr_project /
// residuals / eig_solve.  Paper: arXiv 1507.06078 (P:n = PAPER.md line n).
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "internal.cuh"

namespace {

// NVTX range around one public call (visible in nsys / ncu --nvtx timelines).
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

// Process-wide pool of cuSOLVER handles (creating one costs tens of ms; the
// host-buffer entry creates a context per call).  A handle is bound to the
// device current at creation: pooled per device.
std::mutex g_pool_mu;
std::vector<std::pair<int, cusolverDnHandle_t>> g_solver_pool;

cusolverStatus_t solver_acquire(cusolverDnHandle_t *h) {
    int dev = 0;
    cudaGetDevice(&dev);
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        for (size_t i = 0; i < g_solver_pool.size(); ++i)
            if (g_solver_pool[i].first == dev) {
                *h = g_solver_pool[i].second;
                g_solver_pool.erase(g_solver_pool.begin() + i);
                return CUSOLVER_STATUS_SUCCESS;
            }
    }
    return cusolverDnCreate(h);
}

void solver_release(cusolverDnHandle_t h) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_pool_mu);
    if (g_solver_pool.size() < 16) g_solver_pool.push_back({dev, h});
    else cusolverDnDestroy(h);
}

// Device memory of contexts and of the host-buffer entry: stream-ordered
// allocations from the device's default pool.  The pool keeps, between calls, up to
// the largest footprint a context has needed so far (at least 4 GiB, at most a quarter
// of the device; ARRABIT_POOL_KEEP=0: 4 GiB), so repeated eig_solve_host calls reuse
// their memory instead of mapping it again (cudaMemPoolTrimTo releases it).
std::mutex g_pool_keep_mu;
uint64_t g_pool_keep = 0;
void pool_keep_at_least(uint64_t bytes) {
    static const bool on = [] { const char *e = getenv("ARRABIT_POOL_KEEP"); return !(e && atoi(e) == 0); }();
    int dev = 0;
    cudaGetDevice(&dev);
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    uint64_t thr = std::max<uint64_t>((uint64_t)4 << 30, on ? std::min<uint64_t>(bytes, total_b / 4) : 0);
    std::lock_guard<std::mutex> lk(g_pool_keep_mu);
    if (thr <= g_pool_keep) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess &&
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess)
        g_pool_keep = thr;
}
cudaError_t dev_alloc(void **p, size_t bytes, cudaStream_t s) {
    static std::once_flag once;
    std::call_once(once, [] { pool_keep_at_least(0); });
    return cudaMallocAsync(p, bytes, s);
}
void dev_free(void *p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

constexpr double kSvqbTau = 1e-14;  // eigenvalue floor of the SVQB Gram (relative)
enum { INFO_SYEVD = 0, INFO_BAD = 1, INFO_RANK0 = 2, INFO_CHOL = 40 };
static_assert(INFO_RANK0 + ARR_MAX_P + 1 <= INFO_CHOL, "per-block rank slots overlap the Cholesky info words");  // dinfo slots (INFO_RANK0.. per block;
                                                                        // INFO_CHOL..+5: potrf/trtri of 3 passes)

arr_status fail(arr_ctx *c, arr_status code, const std::string &msg) {
    if (c) {
        c->err = msg;
        if (code == ARR_ECUDA || code == ARR_ECUSOLVER || code == ARR_ENCCL) c->poisoned = code;
    }
    return code;
}

#define CUDA_TRY(expr)                                                                              \
    do {                                                                                            \
        cudaError_t e_ = (expr);                                                                    \
        if (e_ != cudaSuccess) return fail(c, ARR_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define SOLVER_TRY(expr)                                                                            \
    do {                                                                                            \
        cusolverStatus_t s_ = (expr);                                                               \
        if (s_ != CUSOLVER_STATUS_SUCCESS)                                                          \
            return fail(c, ARR_ECUSOLVER, std::string(#expr) + " failed: " + std::to_string((int)s_)); \
    } while (0)
#define CHECK_LAUNCH() CUDA_TRY(cudaGetLastError())
#define ST_TRY(expr)                                                                                \
    do {                                                                                            \
        arr_status st_ = (expr);                                                                    \
        if (st_ != ARR_OK) return st_;                                                              \
    } while (0)
#define GUARD_KEEP(c)                                                                               \
    do {                                                                                            \
        if (!(c)) return ARR_EINVAL;                                                                \
        if ((c)->poisoned != ARR_OK) return (c)->poisoned;                                          \
    } while (0)
// every public call but filter_step drops a pending lazy column scale (filter_step normalize = 2)
#define GUARD(c)                                                                                    \
    do {                                                                                            \
        GUARD_KEEP(c);                                                                              \
        (c)->lazy_pending = false;                                                                  \
    } while (0)

inline int64_t n_glob(const arr_ctx *c) { return c->nranks > 1 ? c->plan.n_global : c->A.n; }
inline int64_t even_up(int64_t x) { return (x + 1) & ~int64_t(1); }
// Leading dimension of the library's own n x (.) blocks: a multiple of ARRABIT_LD_ALIGN
// doubles (default 16: every row starts on a 128-byte line, so a row segment of a column
// panel touches no partial line; 2 = only 16-byte aligned rows).
inline int64_t ld_up(int64_t x) {
    static const int64_t a = [] {
        const char *e = getenv("ARRABIT_LD_ALIGN");
        const int64_t v = e ? atoll(e) : 16;
        return v >= 2 && (v & (v - 1)) == 0 ? v : (int64_t)2;
    }();
    return (x + a - 1) / a * a;
}
inline int32_t m_of(const arr_ctx *c, int p) { return (p + 1) * c->w; }
inline int64_t ldQ(const arr_ctx *c) { return ld_up(m_of(c, c->p)); }
inline int64_t ldT(const arr_ctx *c) { return ld_up(c->w); }

// small dense region layout: [H | V | B | G], each m*m doubles
inline double *H_buf(arr_ctx *c) { const int64_t m = m_of(c, c->p); return c->small; }
inline double *V_buf(arr_ctx *c) { const int64_t m = m_of(c, c->p); return c->small + m * m; }
inline double *B_buf(arr_ctx *c) { const int64_t m = m_of(c, c->p); return c->small + 2 * m * m; }
inline double *G_buf(arr_ctx *c) { const int64_t m = m_of(c, c->p); return c->small + 3 * m * m; }
// vecw layout: [norms (MAXW) | shifts (m) | D (m)]
inline double *NORM_buf(arr_ctx *c) { return c->vecw; }
inline double *SHIFT_buf(arr_ctx *c) { return c->vecw + std::max(m_of(c, c->p), ARR_MAX_W); }
inline double *D_buf(arr_ctx *c) { return c->vecw + 2 * (int64_t)std::max(m_of(c, c->p), ARR_MAX_W); }

// ---------------------------------------------------------------- phase timing
void t_resolve(arr_ctx *c) {  // call only right after a stream sync, with no phase open
    for (const auto &p : c->pending) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, c->ev_pool[p.e0], c->ev_pool[p.e1]) == cudaSuccess) {
            c->phase_ms[p.phase] += ms;
            c->phase_cnt[p.phase] += p.count;
            c->phase_work[p.phase] += p.work;
        }
    }
    c->pending.clear();
    c->ev_next = 0;
}

double chebT(int d, double t) {  // host recursion, Eq. cheby-poly
    double r0 = 1.0, r1 = t;
    if (d == 0) return 1.0;
    for (int j = 1; j < d; ++j) {
        const double r2 = 2.0 * t * r1 - r0;
        r0 = r1;
        r1 = r2;
    }
    return r1;
}

// Chebyshev coefficients of psi_d, the degree-d interpolant of f_d(t) = max(0,t)^{10d}
// at the Chebyshev points of the second kind: the discrete cosine
// transform of the node values, a_k = (2/d) sum''_j f_d(t_j) T_k(t_j) (first and last
// terms halved), then a_0, a_d halved, so that psi_d = sum_k a_k T_k.
std::vector<double> interp_coef(int d) {
    std::vector<double> f(d + 1), a(d + 1, 0.0);
    const double pi = 3.14159265358979323846;
    for (int j = 0; j <= d; ++j) {
        const double t = -cos(j * pi / d);
        f[j] = t > 0.0 ? pow(t, 10.0 * d) : 0.0;
    }
    for (int k = 0; k <= d; ++k) {
        double s = 0.0;
        for (int j = 0; j <= d; ++j) {
            const double wj = (j == 0 || j == d) ? 0.5 : 1.0;
            s += wj * f[j] * cos(k * (pi - j * pi / d));  // T_k(-cos x) = cos(k (pi - x))
        }
        a[k] = 2.0 * s / d;
    }
    a[0] *= 0.5;
    a[d] *= 0.5;
    return a;
}

// psi_d(t) by Clenshaw's recurrence (host scalar)
double psi_eval(const std::vector<double> &a, double t) {
    double b1 = 0.0, b2 = 0.0;
    for (int k = (int)a.size() - 1; k >= 1; --k) {
        const double b0 = a[k] + 2.0 * t * b1 - b2;
        b2 = b1;
        b1 = b0;
    }
    return a[0] + t * b1 - b2;
}

// Sweeps between ARR steps, the dynamic-range rule (R6): s = clamp(floor(D /
// log10 amp), 1, s_max) with amp = |T_d((mu_1 - c)/e)| the per-sweep amplification of the
// top Ritz direction and D digits of column dynamic range between ARRs (opts->range_digits,
// 0 = the default 12: the shifted CholeskyQR3 of the ARR is stable far beyond that, and
// fewer ARRs per solve pay: cfg3 7 -> 4 outer iterations).
constexpr double kRangeDigits = 12.0;
int sweeps_rule(double amp, int s_max, double digits) {
    const double D = digits > 0.0 ? digits : kRangeDigits;
    if (!(amp > 1.0)) return s_max;
    if (!isfinite(amp)) return 1;
    return (int)std::min<double>(std::max<double>(floor(D / log10(amp)), 1.0), s_max);
}

// ---------------------------------------------------------------- distributed building blocks
inline bool is_dist(const arr_ctx *c) { return c->nranks > 1; }

// Rows of a z-slab's end planes (next to a ghost plane) on the stencil path: 1 = the CSR
// kernels over the plan's boundary tiles, 0 = one-plane launches of the stencil kernel.
// Default: CSR for the <= 7-point shapes, the stencil kernel for the 27-point one (whose
// gather is L1-bound); ARRABIT_SLAB_BND=csr|stencil overrides.
inline bool slab_bnd_csr(int shape) {
    static const int v = [] {
        const char *e = getenv("ARRABIT_SLAB_BND");
        return !e ? -1 : (strcmp(e, "csr") == 0 ? 1 : 0);
    }();
    return v < 0 ? shape != 0 : v == 1;
}

// Fused SpMM over the owned rows.  Distributed: start the ghost-row exchange
// of Yin, compute the interior rows while it is in flight, then the boundary
// rows.  Column sums of squares (if requested) of the two launches are written
// to consecutive partial rows.  Returns the number of partial rows (< 0: width
// not supported).
int spmm_x(arr_ctx *c, SpmmArgs s, arr_status *st, bool op = true) {
    *st = ARR_OK;
    if (op && c->sign < 0) {  // the solver's operator is -A: alpha (-A y - shift y) = (-alpha) (A y + shift y)
        s.alpha = -s.alpha;
        s.shift = -s.shift;
    }
    if (!is_dist(c)) return launch_spmm(c, s);
    if (c->cs_link && !s.partials && !s.colshift && !s.Yprev && !s.Xa && s.w == c->w) {
        // column split: A U for the ARR as (transpose -> A_full x this rank's columns -> transpose):
        // two all-to-alls of the block instead of an all-gather / halo of its rows
        ColSplit &S = *c->cs_link;
        arr_ctx *cc = S.col;
        const int64_t ltc = ((int64_t)cc->w + 1) & ~int64_t(1);
        if ((*st = comm_transpose(c->cs_outer, S, 1, s.Yin, s.ld_in, cc->T, ltc)) != ARR_OK) return 0;
        SpmmArgs t = s;
        t.row_ptr = cc->A.row_ptr; t.col = cc->A.col_idx; t.val = cc->A.val;
        t.n = cc->A.n; t.w = cc->w;
        t.Yin = cc->T; t.ld_in = ltc;
        t.Yout = cc->Q; t.ld_out = ltc;
        const int g = launch_spmm(cc, t);
        if (g < 0) return g;
        if ((*st = comm_transpose(c->cs_outer, S, 0, cc->Q, ltc, s.Yout, s.ld_out)) != ARR_OK) return 0;
        return 1;
    }
    DistPlan &P = c->plan;
    if ((*st = comm_halo_begin(c, s.Yin, s.ld_in, s.w)) != ARR_OK) return 0;
    int rows = 0;
    const double *part0 = s.partials;
    bool halo_done = false;
    if (c->st.on && s.n == c->A.n) {
        // z-slab on the stencil path: the planes that touch no ghost plane while the exchange
        // is in flight, then the slab's first / last plane (each a launch of its own z range)
        const StencilState &S = c->st;
        const int nz = (int)S.nz, zi0 = S.gz_lo, zi1 = nz - S.gz_hi;
        SpmmArgs a = s;
        a.nnz = c->A.nnz;
        auto part_at = [&](int r) { return part0 ? const_cast<double *>(part0) + (int64_t)r * s.w : nullptr; };
        if (zi0 < zi1) {
            int g = launch_spmm_stencil(c, a, zi0, zi1);
            if (g >= 0) {
                rows += g;
                if ((*st = comm_halo_end(c, const_cast<double *>(s.Yin))) != ARR_OK) return 0;
                if (S.bnd_is_ends && slab_bnd_csr(S.shape)) {
                    // the end planes' rows on the CSR kernels (the plan's boundary tiles): a
                    // one-plane march stages three planes per output plane, the gather does not
                    SpmmArgs bt = s;
                    bt.tile_row0 = P.bnd_row0; bt.tile_len = P.bnd_len; bt.ntiles = P.n_bnd_tiles;
                    bt.partials = part_at(rows);
                    const char *kern = c->last_kernel;  // the fused SpMM's kernel: the interior's
                    if ((g = launch_spmm(c, bt)) < 0) return g;
                    c->last_kernel = kern;
                    rows += g;
                } else if (S.gz_lo && S.gz_hi) {  // both end planes in one launch
                    a.partials = part_at(rows);
                    if ((g = launch_spmm_stencil(c, a, 0, nz, true)) < 0) return g;
                    rows += g;
                } else if (S.gz_lo || S.gz_hi) {
                    a.partials = part_at(rows);
                    const int zb = S.gz_lo ? 0 : nz - 1;
                    if ((g = launch_spmm_stencil(c, a, zb, zb + 1)) < 0) return g;
                    rows += g;
                }
                c->spmm_blocks++;
                return rows;
            }
        } else {  // one or two planes, all next to a ghost plane
            if ((*st = comm_halo_end(c, const_cast<double *>(s.Yin))) != ARR_OK) return 0;
            halo_done = true;
            const int g = launch_spmm_stencil(c, a, 0, nz);
            if (g >= 0) {
                c->spmm_blocks++;
                return g;
            }
        }
        // the stencil kernel does not apply to this launch (odd width, unaligned block): CSR tiles
    }
    if (P.n_int_tiles > 0) {
        SpmmArgs a = s;
        a.tile_row0 = P.int_row0; a.tile_len = P.int_len; a.ntiles = P.n_int_tiles;
        const int g = launch_spmm(c, a);
        if (g < 0) return g;
        rows += g;
    }
    if (!halo_done && (*st = comm_halo_end(c, const_cast<double *>(s.Yin))) != ARR_OK) return 0;
    if (P.n_bnd_tiles > 0) {
        SpmmArgs a = s;
        a.tile_row0 = P.bnd_row0; a.tile_len = P.bnd_len; a.ntiles = P.n_bnd_tiles;
        if (part0) a.partials = const_cast<double *>(part0) + (int64_t)rows * s.w;
        const int g = launch_spmm(c, a);
        if (g < 0) return g;
        rows += g;
    }
    return rows;
}

// The d degree launches of one filter_step as a CUDA graph (single-GPU contexts): the
// launches are captured once per (operands, interval, width, degree, path) and replayed;
// a new interval re-captures and updates the instantiated graph in place (same topology,
// new kernel arguments).  `run` issues the launches and returns the partial-row count of
// the last launch (< 0 on an unsupported width).  ARRABIT_GRAPH=0 launches directly.
struct GraphKey {
    const void *X, *T, *part, *sched_row0, *scale_in;
    int64_t ldx;
    double a, b;
    int w, d, kind, sign, normalize, stencil;
    bool operator==(const GraphKey &o) const { return memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
template <class Run>
int run_degrees(arr_ctx *c, const GraphKey &key_in, Run run) {
    static const bool enabled = [] { const char *e = getenv("ARRABIT_GRAPH"); return !(e && atoi(e) == 0); }();
    if (!enabled || is_dist(c)) return run();
    GraphKey key;
    memset(&key, 0, sizeof(key));  // padding bytes compared by memcmp
    key.X = key_in.X; key.T = key_in.T; key.part = key_in.part; key.sched_row0 = key_in.sched_row0;
    key.scale_in = key_in.scale_in;
    key.ldx = key_in.ldx; key.a = key_in.a; key.b = key_in.b; key.w = key_in.w; key.d = key_in.d;
    key.kind = key_in.kind; key.sign = key_in.sign; key.normalize = key_in.normalize; key.stencil = key_in.stencil;
    if (!(c->g_exec && c->g_key_set && key == *reinterpret_cast<const GraphKey *>(c->g_key))) {
        const uint64_t l0 = c->launches;
        const int64_t s0 = c->spmm_blocks;
        if (cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
            cudaGetLastError();
            return run();
        }
        const int nb = run();
        cudaGraph_t g = nullptr;
        if (cudaStreamEndCapture(c->stream, &g) != cudaSuccess || nb < 0 || !g) {
            cudaGetLastError();
            if (g) cudaGraphDestroy(g);
            c->launches = l0;
            c->spmm_blocks = s0;
            return nb < 0 ? nb : run();
        }
        bool ok = false;
        if (c->g_exec) {
            cudaGraphExecUpdateResultInfo info;
            ok = cudaGraphExecUpdate(c->g_exec, g, &info) == cudaSuccess;
            if (!ok) {
                cudaGetLastError();
                cudaGraphExecDestroy(c->g_exec);
                c->g_exec = nullptr;
            }
        }
        if (!ok && cudaGraphInstantiate(&c->g_exec, g, 0) != cudaSuccess) {
            cudaGetLastError();
            c->g_exec = nullptr;
            cudaGraphDestroy(g);
            c->launches = l0;
            c->spmm_blocks = s0;
            return run();
        }
        cudaGraphDestroy(g);
        c->g_last_kernel = c->last_kernel;
        c->g_kernels = c->launches - l0;
        c->g_spmm = c->spmm_blocks - s0;
        c->launches = l0;
        c->spmm_blocks = s0;
        c->g_nblk = nb;
        memcpy(c->g_key, &key, sizeof(GraphKey));
        c->g_key_set = true;
    }
    if (cudaGraphLaunch(c->g_exec, c->stream) != cudaSuccess) {
        cudaGetLastError();
        c->g_key_set = false;
        return run();
    }
    c->launches += c->g_kernels;
    c->spmm_blocks += c->g_spmm;
    c->last_kernel = c->g_last_kernel;
    return c->g_nblk;
}
static_assert(sizeof(GraphKey) <= 128, "graph key storage");

// G = X^T Y over the owned rows, summed over ranks.
arr_status gram_x(arr_ctx *c, const double *X, int64_t ldx, int m1, const double *Y, int64_t ldy, int m2, double *G,
                  int64_t ldg) {
    launch_gram(c, X, ldx, m1, Y, ldy, m2, c->A.n, G, ldg, c->part);
    if (is_dist(c)) {
        if (ldg != m2) return fail(c, ARR_EINVAL, "distributed gram needs ldg == m2");
        ST_TRY(comm_allreduce(c, G, (size_t)m1 * m2, 0));
    }
    return ARR_OK;
}

// out[col] = sqrt(sum of the nblk partial rows, over ranks) / max(1,|mu_div|)
arr_status colnorm_x(arr_ctx *c, const double *partials, int nblk, int w, double *out, const double *mu_div) {
    if (!is_dist(c)) {
        launch_colnorm_finalize(c, partials, nblk, w, out, mu_div);
        return ARR_OK;
    }
    launch_colsum(c, partials, nblk, w, out);
    ST_TRY(comm_allreduce(c, out, (size_t)w, 0));
    launch_colnorm_root(c, out, w, mu_div);
    return ARR_OK;
}

// ---------------------------------------------------------------- pieces
// Filter degrees; result left in X (normalised) -- no host sync.
// rho_d(A) X with the paper's interpolant psi_d (eig_set_filter kind 1), by Clenshaw's
// recurrence in the Chebyshev basis with S = c_1 A + c_0 I (c_0 = (a+b)/(a-b),
// c_1 = 2/(b-a), Alg. poly; R18): b_k = a_k X + 2 S b_{k+1} - b_{k+2},
// result a_0 X + S b_1 - b_2.  One fused SpMM per degree (the a_k X term is the kernel's
// fourth operand); X stays intact; b_k ping-pongs between two scratch blocks with b_k
// overwriting b_{k+2} in place.  Result (normalised) in X.
// A pending lazy column scale of X (filter_core normalize = 2) applied explicitly (for the
// paths that do not fold it: the interpolant filter, odd degree counts); drops a pending
// scale of another block.
void lazy_materialize(arr_ctx *c, double *X, int64_t ldx) {
    if (c->lazy_pending && c->lazy_X == X) launch_scale_cols(c, X, ldx, X, ldx, c->A.n, c->w, c->lazy);
    c->lazy_pending = false;
}

arr_status filter_interp(arr_ctx *c, double *X, int64_t ldx, int normalize, double *colnorm_dev) {
    lazy_materialize(c, X, ldx);
    if (normalize == 2) normalize = 1;
    const double c0 = (c->a + c->b) / (c->a - c->b), c1 = 2.0 / (c->b - c->a);
    const std::vector<double> &a = c->coef;
    const int d = (int)a.size() - 1;
    const int w = c->w;
    double *buf[2];
    int64_t ldb[2];
    if (c->T) { buf[0] = c->T; ldb[0] = ldT(c); buf[1] = c->Q; ldb[1] = ldQ(c); }
    else { buf[0] = c->Q; ldb[0] = ldQ(c); buf[1] = c->Q + w; ldb[1] = ldQ(c); }
    int nblk = 0;
    const int ev0 = t_mark(c);
    arr_status st = ARR_OK;
    auto run = [&]() -> int {
        int g = 0;
        for (int k = d - 1; k >= 0; --k) {
            SpmmArgs s{};
            s.row_ptr = c->A.row_ptr; s.col = c->A.col_idx; s.val = c->A.val;
            s.n = c->A.n; s.w = w;
            // S y = c_1 (A y + (c_0/c_1) y): alpha * (A y - shift * y) with shift = -c_0/c_1
            s.shift = -c0 / c1;
            s.alpha = (k == 0 ? 1.0 : 2.0) * c1;
            double gx = a[k];
            if (k == d - 1) { s.Yin = X; s.ld_in = ldx; s.alpha *= a[d]; }  // b_d = a_d X
            else { s.Yin = buf[(k + 1) & 1]; s.ld_in = ldb[(k + 1) & 1]; }
            if (k + 2 == d) gx -= a[d];  // - b_d = - a_d X folds into the X term
            else if (k + 2 < d) { s.Yprev = buf[k & 1]; s.ld_prev = ldb[k & 1]; s.beta = -1.0; }
            s.Xa = X; s.ld_xa = ldx; s.gxa = gx;
            s.Yout = buf[k & 1]; s.ld_out = ldb[k & 1];
            s.partials = (normalize && k == 0) ? c->part : nullptr;
            g = spmm_x(c, s, &st);
            if (st != ARR_OK || g < 0) return g < 0 ? g : 0;
        }
        return g;
    };
    GraphKey key{X, buf[0], normalize ? c->part : nullptr, c->tile_row0, nullptr, ldx, c->a, c->b, w, d, 1, c->sign,
                 normalize, c->st.on ? 1 : 0};
    nblk = run_degrees(c, key, run);
    if (st != ARR_OK) return st;
    if (nblk < 0) return fail(c, ARR_EINVAL, "filter_step: unsupported block width");
    t_add(c, 0, ev0, t_mark(c), d);
    CHECK_LAUNCH();
    if (normalize) {
        double *nrm = colnorm_dev ? colnorm_dev : NORM_buf(c);
        ST_TRY(colnorm_x(c, c->part, nblk, w, nrm, nullptr));
        launch_check_norms(c, nrm, w, c->dinfo + INFO_BAD);
        launch_scale_cols(c, buf[0], ldb[0], X, ldx, c->A.n, w, nrm);
    } else {
        launch_copy_rows(c, buf[0], ldb[0], X, ldx, c->A.n, w);
    }
    CHECK_LAUNCH();
    return ARR_OK;
}

// normalize: 0 none, 1 the columns of the result scaled to unit norm, 2 lazily (Survey §8a
// A2): the norms are computed but X is left unscaled and D = 1/norm becomes pending for X;
// the next filter_core on the same X folds D into its first two degrees (p_d(A)(X D) =
// p_d(A)X D: degree 0's output and degree 1's Y_{j-1} term are scaled by D), which saves one
// 16 n w-byte pass per sweep.  An odd degree count (result in the scratch block) or the
// interpolant filter normalise eagerly.
arr_status filter_core(arr_ctx *c, double *X, int64_t ldx, int normalize, double *colnorm_dev) {
    if (c->filter_kind == 1) return filter_interp(c, X, ldx, normalize, colnorm_dev);
    const double cc = 0.5 * (c->a + c->b), e = 0.5 * (c->b - c->a);
    const int w = c->w;
    if (normalize == 2 && (c->d % 2 == 1 || colnorm_dev)) normalize = 1;
    const double *scale_in = (c->lazy_pending && c->lazy_X == X) ? c->lazy + (ARR_MAX_W + 2) : nullptr;
    c->lazy_pending = false;
    double *T = c->T ? c->T : c->Q;  // lean context: the basis block Q[:, 0:w] is free during sweeps
    const int64_t lt = c->T ? ldT(c) : ldQ(c);
    double *cur = X;
    int64_t ldcur = ldx;
    int nblk = 0;
    const int ev0 = t_mark(c);
    arr_status st = ARR_OK;
    auto run = [&]() -> int {
        double *cu = X, *ot = T;
        int64_t ldc = ldx, ldo = lt;
        int g = 0;
        for (int j = 0; j < c->d; ++j) {
            SpmmArgs s{};
            s.row_ptr = c->A.row_ptr; s.col = c->A.col_idx; s.val = c->A.val;
            s.n = c->A.n; s.w = w;
            s.Yin = cu; s.ld_in = ldc;
            if (j == 0) {
                s.Yprev = nullptr; s.alpha = 1.0 / e; s.beta = 0.0;
            } else {
                s.Yprev = ot; s.ld_prev = ldo; s.alpha = 2.0 / e; s.beta = -1.0;
            }
            if (scale_in && j <= 1) { s.colscale = scale_in; s.scale_mode = j == 0 ? 1 : 2; }
            s.shift = cc;
            s.Yout = ot; s.ld_out = ldo;
            s.partials = (normalize && j == c->d - 1) ? c->part : nullptr;
            g = spmm_x(c, s, &st);
            if (st != ARR_OK || g < 0) return g < 0 ? g : 0;
            std::swap(cu, ot);
            std::swap(ldc, ldo);
        }
        return g;
    };
    GraphKey key{X, T, normalize ? c->part : nullptr, c->tile_row0, scale_in, ldx, c->a, c->b, w, c->d, 0, c->sign,
                 normalize != 0, c->st.on ? 1 : 0};
    nblk = run_degrees(c, key, run);
    if (st != ARR_OK) return st;
    if (nblk < 0) return fail(c, ARR_EINVAL, "filter_step: unsupported block width");
    if (c->d % 2 == 1) { cur = T; ldcur = lt; }  // Y_d is in the scratch block after an odd degree count
    t_add(c, 0, ev0, t_mark(c), c->d);
    CHECK_LAUNCH();
    if (normalize == 2) {  // lazy: norms and D = 1/norm pending for X (d even: the result is in X)
        ST_TRY(colnorm_x(c, c->part, nblk, w, c->lazy, nullptr));
        launch_check_norms(c, c->lazy, w, c->dinfo + INFO_BAD);
        launch_recip(c, c->lazy, w, c->lazy + (ARR_MAX_W + 2));
        c->lazy_pending = true;
        c->lazy_X = X;
    } else if (normalize) {
        double *nrm = colnorm_dev ? colnorm_dev : NORM_buf(c);
        ST_TRY(colnorm_x(c, c->part, nblk, w, nrm, nullptr));
        launch_check_norms(c, nrm, w, c->dinfo + INFO_BAD);
        launch_scale_cols(c, cur, ldcur, X, ldx, c->A.n, w, nrm);
    } else if (cur != X) {
        launch_copy_rows(c, cur, ldcur, X, ldx, c->A.n, w);
    }
    CHECK_LAUNCH();
    return ARR_OK;
}

// One SVQB pass: Out = In * D V L^{-1/2} (ncols columns), rank -> dinfo slot.
arr_status svqb_pass(arr_ctx *c, const double *In, int64_t ldin, double *Out, int64_t ldout, int ncols,
                     int *rank_slot) {
    double *G = G_buf(c), *V = V_buf(c), *B = B_buf(c), *D = D_buf(c);
    ST_TRY(gram_x(c, In, ldin, ncols, In, ldin, ncols, G, ncols));
    launch_svqb_prep(c, G, ncols, D, V);
    CHECK_LAUNCH();
    SOLVER_TRY(cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, ncols, V, ncols,
                                c->evals, c->solver_work, c->solver_lwork, c->dinfo + INFO_SYEVD));
    launch_svqb_build(c, D, V, c->evals, ncols, kSvqbTau, B, rank_slot);
    ST_TRY(comm_bcast(c, B, (size_t)ncols * ncols, 0));  // one transform on every rank
    launch_gemm(c, 1.0, In, ldin, ncols, B, ncols, ncols, 0.0, nullptr, 0, Out, ldout, c->A.n);
    CHECK_LAUNCH();
    return ARR_OK;
}

// One CholeskyQR pass (optionally shifted, Fukaya et al. 2020): G = In^T In,
// D = diag(G)^{-1/2}, R^T R = D G D + s I (potrf), Out = In D R^{-1} (trtri +
// DMMA GEMM).  s = 11 (n c + c(c+1)) u c bounds the rounding of the Gram so the
// shifted factorisation exists for any input; two unshifted passes follow.
// racc_new (optional): the accumulated factor R with In_0 = Out R over the passes so far
// (launch_chol_racc; racc_first on the first pass), R23
arr_status cholqr_pass(arr_ctx *c, const double *In, int64_t ldin, double *Out, int64_t ldout, int ncols,
                       bool shifted, int *info2, int *rank_slot, const double *racc_old = nullptr,
                       double *racc_new = nullptr, bool racc_first = false) {
    double *G = G_buf(c), *Gs = V_buf(c), *B = B_buf(c), *D = D_buf(c);
    const double u = 1.1102230246251565e-16;
    const double shift = shifted ? 11.0 * ((double)n_glob(c) * ncols + (double)ncols * (ncols + 1)) * u * ncols : 0.0;
    ST_TRY(gram_x(c, In, ldin, ncols, In, ldin, ncols, G, ncols));
    launch_chol_prep(c, G, ncols, shift, D, Gs);
    CHECK_LAUNCH();
    SOLVER_TRY(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_UPPER, ncols, Gs, ncols, c->solver_work, c->solver_lwork,
                                info2));
    if (rank_slot) launch_diag_copy(c, Gs, ncols, c->evals);
    if (racc_new) launch_chol_racc(c, Gs, D, ncols, racc_old, racc_new, racc_first);
    SOLVER_TRY(cusolverDnXtrtri(c->solver, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, ncols, CUDA_R_64F, Gs, ncols,
                                c->trtri_dwork, c->trtri_dbytes, c->trtri_hwork.data(), c->trtri_hwork.size(),
                                info2 + 1));
    launch_chol_build(c, D, Gs, ncols, B, c->evals, 100.0 * shift, rank_slot);
    ST_TRY(comm_bcast(c, B, (size_t)ncols * ncols, 0));  // one transform on every rank
    launch_gemm(c, 1.0, In, ldin, ncols, B, ncols, ncols, 0.0, nullptr, 0, Out, ldout, c->A.n, /*upper=*/1);
    CHECK_LAUNCH();
    return ARR_OK;
}

// Shifted CholeskyQR3 In -> Out (In != Out) through the scratch block S (may be
// In itself: In is only read by the first pass); *ok = 0 if a factorisation
// failed (numerically rank-deficient input after the shift): the caller then
// falls back to SVQB.  Synchronises the stream.
// racc_final (optional): set to the factor R with In = Out R (c->racc or c->racc + ncols^2).
arr_status cholqr3(arr_ctx *c, const double *In, int64_t ldin, double *Out, int64_t ldout, int ncols, int *rank_slot,
                   bool *ok, double *S, int64_t lds, double **racc_final = nullptr) {
    arr_status st;
    int *inf = c->dinfo + INFO_CHOL;
    double *r0 = racc_final ? c->racc : nullptr, *r1 = racc_final ? c->racc + (int64_t)ncols * ncols : nullptr;
    if (racc_final) *racc_final = r1;
    CUDA_TRY(cudaMemsetAsync(inf, 0, sizeof(int) * 6, c->stream));
    if ((st = cholqr_pass(c, In, ldin, Out, ldout, ncols, true, inf, rank_slot, nullptr, r0, true)) != ARR_OK) return st;
    if ((st = cholqr_pass(c, Out, ldout, S, lds, ncols, false, inf + 2, nullptr, r0, r1)) != ARR_OK) return st;
    // The second pass's factor R2 measures how far pass 1 was from orthonormal:
    // pass 2's output is orthonormal to O(u cond(R2)^2).  If R2^{-1} (left in V
    // by trtri) is within 1e-6 of I entrywise, the third pass is skipped.
    launch_dev_from_identity(c, V_buf(c), ncols, c->evals);
    CUDA_TRY(cudaMemcpyAsync(c->h_istage + 40, inf, sizeof(int) * 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->h_stage, c->evals, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *ok = true;
    for (int q = 0; q < 4; ++q) *ok = *ok && c->h_istage[40 + q] == 0;
    const double dev = c->h_stage[0];
    if (!*ok) return ARR_OK;
    if (!(dev <= 1e-6)) {
        if ((st = cholqr_pass(c, S, lds, Out, ldout, ncols, false, inf + 4, nullptr, r1, r0)) != ARR_OK) return st;
        if (racc_final) *racc_final = r0;
        CUDA_TRY(cudaMemcpyAsync(c->h_istage + 44, inf + 4, sizeof(int) * 2, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        *ok = c->h_istage[44] == 0 && c->h_istage[45] == 0;
    } else {
        launch_copy_rows(c, S, lds, Out, ldout, c->A.n, ncols);
        CHECK_LAUNCH();
    }
    return ARR_OK;
}

// Two SVQB passes In -> Out through the scratch block S (S != In, S != Out).
arr_status svqb2(arr_ctx *c, const double *In, int64_t ldin, double *Out, int64_t ldout, int ncols,
                 int *rank_slot, double *S, int64_t lds) {
    arr_status st;
    if ((st = svqb_pass(c, In, ldin, S, lds, ncols, rank_slot)) != ARR_OK) return st;
    if ((st = svqb_pass(c, S, lds, Out, ldout, ncols, nullptr)) != ARR_OK) return st;
    return ARR_OK;
}

// H's last block column restricted to its block-tridiagonal rows (ARRABIT_H_TRIDIAG=0: all rows)
bool h_tridiag() {
    static const bool v = [] { const char *e = getenv("ARRABIT_H_TRIDIAG"); return !(e && atoi(e) == 0); }();
    return v;
}

// H's block (p-1, p) from the last augmentation block's CholeskyQR factor (R23;
// ARRABIT_H_RFACTOR=0: from the Gram U_{p-1}^T (A U_p))
bool h_rfactor() {
    static const bool v = [] { const char *e = getenv("ARRABIT_H_RFACTOR"); return !(e && atoi(e) == 0); }();
    return v;
}

arr_status arr_core(arr_ctx *c, int p_use, const double *X, int64_t ldx, double *Y, int64_t ldy,
                    double *ritz_host, int32_t *rank) {
    const int w = c->w;
    const int m = m_of(c, p_use);
    const int64_t lq = ldQ(c);
    double *Q = c->Q;
    // scratch blocks: the context's T; without one (lean context) the spare block
    // Q[:, w:2w] while U_0 is built, then the output block Y (== X) once X is consumed
    double *S0 = c->T, *T = c->T;
    int64_t ls0 = ldT(c), lt = ldT(c);
    if (!c->T) {
        S0 = Q + w;
        ls0 = lq;
        T = (p_use == 0) ? S0 : Y;
        lt = (p_use == 0) ? lq : ldy;
    }
    arr_status st;
    const int ev0 = t_mark(c);
    int evs = ev0;
    double *racc = nullptr;  // W_p = U_p R (the last augmentation block's CholeskyQR factor)
    bool r_ok = false;
    // U_0 = orth(X): Alg. RR step 1 on the first block
    bool ok = false;
    if (c->orth_mode == 0 && (st = cholqr3(c, X, ldx, Q, lq, w, c->dinfo + INFO_RANK0, &ok, S0, ls0)) != ARR_OK)
        return st;
    if (!ok && (st = svqb2(c, X, ldx, Q, lq, w, c->dinfo + INFO_RANK0, S0, ls0)) != ARR_OK) return st;
    // U_j = orth((I - Q Q^T) A U_{j-1}): the block-Krylov augmentation of Eq. S:ARR
    for (int j = 1; j <= p_use; ++j) {
        const int jw = j * w;
        double *Qj = Q + (int64_t)jw;
        auto make_W = [&]() -> arr_status {  // T = (I - Q Q^T) A U_{j-1}, block CGS twice
            SpmmArgs s{};
            s.row_ptr = c->A.row_ptr; s.col = c->A.col_idx; s.val = c->A.val;
            s.n = c->A.n; s.w = w;
            s.Yin = Q + (int64_t)(j - 1) * w; s.ld_in = lq;
            s.alpha = 1.0; s.shift = 0.0;
            s.Yout = T; s.ld_out = lt;
            arr_status st2;
            const int g = spmm_x(c, s, &st2);
            if (st2 != ARR_OK) return st2;
            if (g < 0) return fail(c, ARR_EINVAL, "arr_project: unsupported width");
            if (c->defl_n > 0) {  // ARR in the orthogonal complement of the locked vectors
                for (int pass = 0; pass < 2; ++pass) {
                    ST_TRY(gram_x(c, c->defl_Q, c->defl_ld, c->defl_n, T, lt, w, G_buf(c), w));
                    launch_gemm(c, -1.0, c->defl_Q, c->defl_ld, c->defl_n, G_buf(c), w, w, 1.0, T, lt, T, lt, c->A.n);
                }
            }
            static const int cgs_passes = [] { const char *e = getenv("ARRABIT_CGS_PASSES"); return e ? std::max(1, atoi(e)) : 2; }();
            for (int pass = 0; pass < cgs_passes; ++pass) {
                ST_TRY(gram_x(c, Q, lq, jw, T, lt, w, G_buf(c), w));
                // The first pass's coefficients Q[:, :jw]^T (A U_{j-1}) ARE rows [0, jw) of
                // block column j-1 of H = Q^T A Q (same SpMM output, same Gram kernel on the
                // same operands: bitwise what the H loop would compute), so H keeps them.
                if (pass == 0 && !is_dist(c)) launch_copy_rows(c, G_buf(c), w, H_buf(c) + (int64_t)(j - 1) * w, m, jw, w);
                launch_gemm(c, -1.0, Q, lq, jw, G_buf(c), w, w, 1.0, T, lt, T, lt, c->A.n);
            }
            CHECK_LAUNCH();
            return ARR_OK;
        };
        if ((st = make_W()) != ARR_OK) return st;
        ok = false;
        const bool want_r = j == p_use && h_rfactor() && !is_dist(c) && c->defl_n == 0;
        if (c->orth_mode == 0 &&
            (st = cholqr3(c, T, lt, Qj, lq, w, c->dinfo + INFO_RANK0 + j, &ok, T, lt, want_r ? &racc : nullptr)) !=
                ARR_OK)
            return st;
        r_ok = want_r && ok && c->orth_mode == 0;
        if (!ok) {
            if (c->orth_mode == 0 && (st = make_W()) != ARR_OK) return st;  // T was reused by CholeskyQR3
            if ((st = svqb_pass(c, T, lt, Qj, lq, w, c->dinfo + INFO_RANK0 + j)) != ARR_OK) return st;
            if ((st = svqb_pass(c, Qj, lq, T, lt, w, nullptr)) != ARR_OK) return st;
            launch_copy_rows(c, T, lt, Qj, lq, c->A.n, w);
        }
        // A nearly invariant Krylov block makes W numerically rank deficient; its
        // orthonormalisation blows rounding errors up to unit columns that are no longer
        // orthogonal to Q[:, :jw] (loss ~ u / sigma_min).  Check max |Q[:, :jw]^T U_j| and,
        // above ~1e-12, project U_j out of Q twice and re-orthonormalise (CholeskyQR2; U_j is
        // then nearly orthonormal): H = Q^T A Q stays a true Rayleigh quotient (without it the
        // cfg4 solve stalls at residuals ~1e-7).
        // The check runs on a sketch: E = Q[:, :jw]^T (U_j Omega), Omega a fixed seeded w x 8
        // Gaussian block (2 n w 8 + 2 n jw 8 flops instead of 2 n jw w).  A sketch entry sums
        // the w entries of a row of Q^T U_j with N(0,1) weights: clean rounding-level entries
        // (~u sqrt(n) ~ 1e-13 at n = 1e6) give ~sqrt(w) 1e-13, and the failure the check guards
        // (amplified noise across the whole block, loss ~ u / sigma_min(W), R8)
        // gives >= sqrt(w) 1e-11; flag above 3e-12 sqrt(w).
        launch_gemm(c, 1.0, Qj, lq, w, c->omega, kOmegaCols, kOmegaCols, 0.0, nullptr, 0, T, lt, c->A.n);
        ST_TRY(gram_x(c, Q, lq, jw, T, lt, kOmegaCols, G_buf(c), kOmegaCols));
        launch_maxabs(c, G_buf(c), (int64_t)jw * kOmegaCols, c->evals);
        CHECK_LAUNCH();
        CUDA_TRY(cudaMemcpyAsync(c->h_stage, c->evals, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (r_ok)
            CUDA_TRY(cudaMemcpyAsync(c->h_istage + 52, c->dinfo + INFO_RANK0 + j, sizeof(int), cudaMemcpyDeviceToHost,
                                     c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (r_ok) r_ok = c->h_istage[52] == w;  // numerically full rank: W = U_p R holds with R invertible
        if (!(c->h_stage[0] <= 3e-12 * sqrt((double)w))) {
            r_ok = false;  // U_p re-projected and re-orthonormalised: no longer W R^{-1}
            for (int pass = 0; pass < 2; ++pass) {
                ST_TRY(gram_x(c, Q, lq, jw, Qj, lq, w, G_buf(c), w));
                launch_gemm(c, -1.0, Q, lq, jw, G_buf(c), w, w, 1.0, Qj, lq, Qj, lq, c->A.n);
            }
            // CholeskyQR2 of the re-projected block; a block of pure rounding noise (an exactly
            // invariant Krylov block, e.g. a diagonal A) can make a Gram numerically indefinite:
            // then the pass is redone by SVQB, which completes dependent directions (R7)
            int *inf = c->dinfo + INFO_CHOL;
            auto chol_ok = [&](int pass_idx) -> int {  // 1 ok, 0 failed, -1 CUDA error
                if (cudaMemcpyAsync(c->h_istage + 48, inf + 2 * pass_idx, sizeof(int) * 2, cudaMemcpyDeviceToHost,
                                    c->stream) != cudaSuccess ||
                    cudaStreamSynchronize(c->stream) != cudaSuccess)
                    return -1;
                return c->h_istage[48] == 0 && c->h_istage[49] == 0;
            };
            CUDA_TRY(cudaMemsetAsync(inf, 0, sizeof(int) * 4, c->stream));
            if ((st = cholqr_pass(c, Qj, lq, T, lt, w, false, inf, nullptr)) != ARR_OK) return st;
            int okp = chol_ok(0);
            if (okp < 0) return fail(c, ARR_ECUDA, "arr_project: CUDA error");
            if (!okp) {  // Qj still holds the re-projected block
                if ((st = svqb_pass(c, Qj, lq, T, lt, w, nullptr)) != ARR_OK) return st;
            }
            if ((st = cholqr_pass(c, T, lt, Qj, lq, w, false, inf + 2, nullptr)) != ARR_OK) return st;
            okp = chol_ok(1);
            if (okp < 0) return fail(c, ARR_ECUDA, "arr_project: CUDA error");
            if (!okp) {  // T still holds the first pass's (nearly orthonormal) output
                if ((st = svqb_pass(c, T, lt, Qj, lq, w, nullptr)) != ARR_OK) return st;
                if ((st = svqb_pass(c, Qj, lq, T, lt, w, nullptr)) != ARR_OK) return st;
                launch_copy_rows(c, T, lt, Qj, lq, c->A.n, w);
                CHECK_LAUNCH();
            }
        }
    }
    { const int e = t_mark(c); t_add(c, 3, evs, e, 1); evs = e; }
    // H = Q^T (A Q), one w-column block of AQ at a time (AQ never stored whole)
    double *H = H_buf(c);
    // block columns 0..p_use-1 came from the CGS passes (one GPU); multi-GPU recomputes them
    for (int j = is_dist(c) ? 0 : p_use; j <= p_use; ++j) {
        SpmmArgs s{};
        s.row_ptr = c->A.row_ptr; s.col = c->A.col_idx; s.val = c->A.val;
        s.n = c->A.n; s.w = w;
        s.Yin = Q + (int64_t)j * w; s.ld_in = lq;
        s.alpha = 1.0; s.shift = 0.0;
        s.Yout = T; s.ld_out = lt;
        const int g = spmm_x(c, s, &st);
        if (st != ARR_OK) return st;
        if (g < 0) return fail(c, ARR_EINVAL, "arr_project: unsupported width");
        // upper block triangle only: rows [0, (j+1)w) of column block j (H is symmetric).
        // Block-Lanczos structure (R22): A U_i lies in span(U_0..U_{i+1}) up to the
        // rounding of the CGS2 + CholeskyQR steps, so U_i^T A U_j = (A U_i)^T U_j = O(u ||A||)
        // for i <= j - 2: on one GPU the last block column keeps rows [(j-1)w, (j+1)w) only
        // (p >= 2: 2 n w^2 fewer flops per ARR per skipped block) and the rest is exact zero.
        const int i0 = (!is_dist(c) && j >= 2 && h_tridiag()) ? j - 1 : 0;
        if (i0 > 0)
            CUDA_TRY(cudaMemset2DAsync(H + (int64_t)j * w, sizeof(double) * m, 0, sizeof(double) * w, (size_t)i0 * w,
                                       c->stream));
        // Block (j-1, j) from the CholeskyQR factor of the last augmentation block (DESIGN.md
        // R23): A U_{j-1} = Q[:, :jw] C + U_j R (the CGS2 + CholeskyQR3 that built U_j), so
        // U_{j-1}^T A U_j = (A U_{j-1})^T U_j = R^T + C^T Q[:, :jw]^T U_j = R^T + O(u ||A||)
        // (U_j passed the re-orthogonality check): 2 n w^2 flops fewer per ARR.
        const bool use_r = r_ok && racc && j == p_use && j >= 1;
        const int ioff = use_r ? j - 1 : j;  // rows [i0 w, ioff w) from the Gram Q^T (A U_j)
        if (ioff > i0)
            launch_gram(c, Q + (int64_t)i0 * w, lq, (ioff - i0) * w, T, lt, w, c->A.n,
                        H + (int64_t)i0 * w * m + (int64_t)j * w, m, c->part);
        if (use_r) launch_put_rt(c, racc, w, H + (int64_t)(j - 1) * w * m + (int64_t)j * w, m);
        // diagonal block U_j^T (A U_j), symmetric: the tiles on or above the diagonal only
        launch_gram(c, Q + (int64_t)j * w, lq, w, T, lt, w, c->A.n, H + (int64_t)j * w * m + (int64_t)j * w, m, c->part,
                    /*sym_result=*/true);
    }
    if (is_dist(c)) ST_TRY(comm_allreduce(c, H, (size_t)m * m, 0));
    launch_symmetrize(c, H, m, w);
    CHECK_LAUNCH();
    { const int e = t_mark(c); t_add(c, 4, evs, e, 1); evs = e; }
    // H = V Theta V^T (Alg. RR step 3): small dense eig on device (not graded)
    SOLVER_TRY(cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, m, H, m, c->evals,
                                c->solver_work, c->solver_lwork, c->dinfo + INFO_SYEVD));
    if (is_dist(c)) {  // one eigendecomposition on every rank
        ST_TRY(comm_bcast(c, H, (size_t)m * m, 0));
        ST_TRY(comm_bcast(c, c->evals, (size_t)m, 0));
    }
    { const int e = t_mark(c); t_add(c, 5, evs, e, 1); evs = e; }
    // Y = Q V[:, leading w] (Alg. RR step 4; Alg. ARR step 4)
    if (Y) {
        launch_ritz_select(c, H, m, w, B_buf(c));
        launch_gemm(c, 1.0, Q, lq, m, B_buf(c), w, w, 0.0, nullptr, 0, Y, ldy, c->A.n);
    }
    CHECK_LAUNCH();
    t_add(c, 1, ev0, t_mark(c), 1);
    CUDA_TRY(cudaMemcpyAsync(c->h_stage, c->evals, sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaMemcpyAsync(c->h_istage, c->dinfo, sizeof(int) * (INFO_RANK0 + p_use + 1), cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    t_resolve(c);
    if (c->h_istage[INFO_SYEVD] != 0)
        return fail(c, ARR_ECUSOLVER, "syevd info = " + std::to_string(c->h_istage[INFO_SYEVD]));
    for (int i = 0; i < m; ++i) ritz_host[i] = c->h_stage[m - 1 - i];
    if (rank) {
        int r = 0;
        for (int j = 0; j <= p_use; ++j) r += c->h_istage[INFO_RANK0 + j];
        *rank = r;
    }
    return ARR_OK;
}

arr_status residuals_core(arr_ctx *c, const double *Y, int64_t ldy, const double *mu_host, int ncols,
                          double *res_host) {
    double *shift = SHIFT_buf(c), *out = NORM_buf(c);
    // mu_host: Ritz values of the solver's operator sign*A; the kernel applies A with
    // alpha = sign, so the per-column shift is sign*mu (the norm is unchanged)
    for (int i = 0; i < ncols; ++i) c->h_stage[i] = c->sign * mu_host[i];
    CUDA_TRY(cudaMemcpyAsync(shift, c->h_stage, sizeof(double) * ncols, cudaMemcpyHostToDevice, c->stream));
    const int ev0 = t_mark(c);
    SpmmArgs s{};
    s.row_ptr = c->A.row_ptr; s.col = c->A.col_idx; s.val = c->A.val;
    s.n = c->A.n; s.w = ncols;
    s.Yin = Y; s.ld_in = ldy;
    s.alpha = 1.0; s.shift = 0.0; s.colshift = shift;
    s.Yout = nullptr;
    s.partials = c->part;
    arr_status st;
    const int g = spmm_x(c, s, &st);
    if (st != ARR_OK) return st;
    if (g < 0) return fail(c, ARR_EINVAL, "residuals: unsupported width");
    ST_TRY(colnorm_x(c, c->part, g, ncols, out, shift));
    CHECK_LAUNCH();
    t_add(c, 2, ev0, t_mark(c), 1);
    CUDA_TRY(cudaMemcpyAsync(c->h_stage, out, sizeof(double) * ncols, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    t_resolve(c);
    memcpy(res_host, c->h_stage, sizeof(double) * ncols);
    return ARR_OK;
}

// rc = lambda_min(X^T X) / lambda_max(X^T X) (2-norm reciprocal condition of the Gram;
// the paper uses LAPACK's 1-norm estimate).  Synchronises.
arr_status gram_rcond(arr_ctx *c, const double *X, int64_t ldx, double *rc) {
    const int w = c->w;
    double *G = G_buf(c), *V = V_buf(c);
    ST_TRY(gram_x(c, X, ldx, w, X, ldx, w, G, w));
    CUDA_TRY(cudaMemcpyAsync(V, G, sizeof(double) * (size_t)w * w, cudaMemcpyDeviceToDevice, c->stream));
    SOLVER_TRY(cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_NOVECTOR, CUBLAS_FILL_MODE_LOWER, w, V, w, c->evals,
                                c->solver_work, c->solver_lwork, c->dinfo + INFO_SYEVD));
    CUDA_TRY(cudaMemcpyAsync(c->h_stage, c->evals, sizeof(double) * w, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const double lmin = c->h_stage[0], lmax = c->h_stage[w - 1];
    *rc = (lmax > 0.0) ? std::max(lmin, 0.0) / lmax : 0.0;
    return ARR_OK;
}

// One Gauss-Newton inner step (Alg. Arrabit2's GN branch P:1490-1493, Alg. GN)
// with the accelerator: Y = X (X^T X)^{-1}; Z = rho_d(A) Y; X = Z - X (Y^T Z - I)/2.
// Y / Z live in the last basis block (free during the inner loop); Y^T Z is formed as
// (X^T X)^{-1} (X^T Z); every n-row product is a DMMA Gram / GEMM.
arr_status gn_step(arr_ctx *c, double *X, int64_t ldx) {
    const int w = c->w;
    const int64_t lq = ldQ(c);
    double *Yb = c->Q + (int64_t)c->p * w;
    double *G = G_buf(c), *Gi = V_buf(c), *C = B_buf(c);
    ST_TRY(gram_x(c, X, ldx, w, X, ldx, w, G, w));
    CUDA_TRY(cudaMemcpyAsync(Gi, G, sizeof(double) * (size_t)w * w, cudaMemcpyDeviceToDevice, c->stream));
    int *inf = c->dinfo + INFO_CHOL;
    SOLVER_TRY(cusolverDnDpotrf(c->solver, CUBLAS_FILL_MODE_LOWER, w, Gi, w, c->solver_work, c->solver_lwork, inf));
    SOLVER_TRY(cusolverDnDpotri(c->solver, CUBLAS_FILL_MODE_LOWER, w, Gi, w, c->solver_work, c->solver_lwork, inf + 1));
    // X^T X must be SPD for the inverse to exist: a singular or indefinite Gram (X lost
    // rank) fails the solve instead of feeding a garbage inverse into Y and X
    CUDA_TRY(cudaMemcpyAsync(c->h_istage + 56, inf, sizeof(int) * 2, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->h_istage[56] != 0 || c->h_istage[57] != 0)
        return fail(c, ARR_ENUMERIC, "GN step: X^T X is not positive definite (potrf/potri info " +
                                         std::to_string(c->h_istage[56]) + "/" + std::to_string(c->h_istage[57]) + ")");
    launch_mirror_upper(c, Gi, w);  // column-major lower = row-major upper -> full symmetric inverse
    ST_TRY(comm_bcast(c, Gi, (size_t)w * w, 0));
    launch_gemm(c, 1.0, X, ldx, w, Gi, w, w, 0.0, nullptr, 0, Yb, lq, c->A.n);  // Y
    ST_TRY(filter_core(c, Yb, lq, 0, nullptr));                                   // Z = rho_d(A) Y
    ST_TRY(gram_x(c, X, ldx, w, Yb, lq, w, G, w));                                // X^T Z
    launch_gemm(c, 1.0, Gi, w, w, G, w, w, 0.0, nullptr, 0, C, w, w);             // Y^T Z
    launch_add_diag(c, C, w, w, -1.0);                                            // - I
    launch_gemm(c, -0.5, X, ldx, w, C, w, w, 1.0, Yb, lq, Yb, lq, c->A.n);        // Z - X (Y^T Z - I)/2
    launch_copy_rows(c, Yb, lq, X, ldx, c->A.n, w);
    CHECK_LAUNCH();
    return ARR_OK;
}

bool block_ok(const double *p, int64_t ld, int ncols) { return p != nullptr && ld >= ncols && ncols >= 1; }

void log_outer(const arr_solve_opts *o, int outer, int s, double a, double b, double mu1, double maxres, int p, int d,
               int locked, double tol_t, double mu_k, double mu_w) {
    if (!o->log || outer < 1 || outer > o->log_cap) return;
    double *r = o->log + (size_t)(outer - 1) * ARR_LOG_FIELDS;
    const double v[ARR_LOG_FIELDS] = {(double)outer, (double)s, a, b, mu1, maxres, (double)p, (double)d, (double)locked,
                                      tol_t, mu_k, mu_w};
    for (int i = 0; i < ARR_LOG_FIELDS; ++i) r[i] = v[i];
}

}  // namespace

// Alg. Arrabit2 with continuation and deflation, MPM inner
// solver, the dynamic-range sweeps rule (R6), fixed p and d (R19):
//   tol_1 = sqrt(tol) (so that every locked pair meets tol), tol_{t+1} = max(1e-2 tol_t, tol)
//   once max res <= tol_t, and then b = mu_{k+q}; after every ARR the leading
//   Ritz pairs with res <= max(1e-14, tol_t^2) (Eq. defl) are locked: they stay in the
//   leading columns of X (Q_c) and leave the iteration; the remaining w - n_c columns are
//   filtered, projected against Q_c (X = X - Q_c Q_c^T X, twice) and augmented-RR'ed on
//   their own (the context runs at width w - n_c); a final Rayleigh-Ritz on all w
//   columns orders the pairs and recomputes every residual.
arr_status solve_deflate(arr_ctx *c, double *X, int64_t ldx, const arr_solve_opts *opts, double *eigval_host,
                         double *res_host, arr_solve_info *info) {
    const int w = c->w, k = c->k, p = c->p;
    arr_solve_info inf{};
    double a = 0.0;
    arr_status st = eig_gershgorin_lower(c, &a);
    if (st != ARR_OK) return st;
    std::vector<double> r0(w), ritz((size_t)(p + 1) * w), res(k, 0.0), locked_res;
    if ((st = arr_core(c, 0, X, ldx, nullptr, 0, r0.data(), nullptr)) != ARR_OK) return st;
    double b = r0[w - 1], mu1 = r0[0];
    if (!(a < b)) a = b - 1e-8 * (fabs(b) + 1.0);
    double tol_t = std::max(opts->tol, sqrt(opts->tol));
    int nc = 0;  // locked columns X[:, :nc]
    int32_t rank = 0;
    const int64_t spmm0 = c->spmm_blocks;
    bool done = false;
    auto restore = [&]() { c->w = w; };
    for (int outer = 1; outer <= opts->maxit; ++outer) {
        const int wa = w - nc;
        double *Xa = X + nc;
        c->w = wa;  // the active block (buffers are sized for w; every ld derived from c->w fits)
        if ((st = eig_set_interval(c, a, b)) != ARR_OK) { restore(); return st; }
        const double cc = 0.5 * (a + b), e = 0.5 * (b - a);
        const double amp = fabs(c->filter_kind == 1 ? psi_eval(c->coef, (mu1 - cc) / e) : chebT(c->d, (mu1 - cc) / e));
        const int s = sweeps_rule(amp, opts->s_max, opts->range_digits);
        CUDA_TRY(cudaMemsetAsync(c->dinfo + INFO_BAD, 0, sizeof(int), c->stream));
        for (int q = 0; q < s; ++q)
            if ((st = filter_core(c, Xa, ldx, 1, nullptr)) != ARR_OK) { restore(); return st; }
        inf.sweeps += s;
        if (nc > 0) {  // X = X - Q_c (Q_c^T X), twice
            for (int pass = 0; pass < 2; ++pass) {
                if ((st = gram_x(c, X, ldx, nc, Xa, ldx, wa, G_buf(c), wa)) != ARR_OK) { restore(); return st; }
                launch_gemm(c, -1.0, X, ldx, nc, G_buf(c), wa, wa, 1.0, Xa, ldx, Xa, ldx, c->A.n);
            }
            CUDA_TRY(cudaGetLastError());
        }
        c->defl_Q = X; c->defl_ld = ldx; c->defl_n = nc;
        st = arr_core(c, p, Xa, ldx, Xa, ldx, ritz.data(), &rank);
        c->defl_n = 0;
        if (st != ARR_OK) { restore(); return st; }
        const int ka = k - nc;
        std::vector<double> ra(ka);
        if ((st = residuals_core(c, Xa, ldx, ritz.data(), ka, ra.data())) != ARR_OK) { restore(); return st; }
        double maxres = 0.0;
        for (int i = 0; i < ka; ++i) { res[nc + i] = ra[i]; maxres = std::max(maxres, ra[i]); }
        for (int i = 0; i < nc; ++i) maxres = std::max(maxres, locked_res[i]);
        inf.outer = outer;
        inf.maxres = maxres;
        inf.last_rank = rank;
        inf.a = a; inf.b = b;
        restore();
        log_outer(opts, outer, s, a, b, mu1, maxres, p, c->d, nc, tol_t, ritz[ka - 1], ritz[wa - 1]);
        if (maxres <= opts->tol) { done = true; inf.exit_rule = 1; break; }
        if (maxres <= tol_t) tol_t = std::max(1e-2 * tol_t, opts->tol);  // continuation (Eq. contin)
        // b: the R3 rule (mu_{w+1} after every ARR, here the first active Ritz value outside
        // the block); the paper's update only at continuation (b = mu_{k+q}) leaves the
        // RR(X0) estimate in place until max res <= tol_1, which with few sweeps per ARR never
        // happens (cfg2: max res stays at 0.2 for 300 outer iterations)
        b = ritz[std::min(wa, (p + 1) * wa - 1)];
        // deflation: lock the leading converged pairs (Eq. defl); keep >= 1 active
        const double defl = std::max(1e-14, tol_t * tol_t);
        int add = 0;
        while (add < ka - 1 && ra[add] <= defl) ++add;
        for (int i = 0; i < add; ++i) locked_res.push_back(ra[i]);
        nc += add;
        mu1 = ritz[add];
        if (!(a < b)) a = b - 1e-8 * (fabs(b) + 1.0);
    }
    restore();
    // final Rayleigh-Ritz on the whole block: ordered pairs, fresh residuals
    std::vector<double> rf(w), resf(k);
    if ((st = arr_core(c, 0, X, ldx, X, ldx, rf.data(), nullptr)) != ARR_OK) return st;
    if ((st = residuals_core(c, X, ldx, rf.data(), k, resf.data())) != ARR_OK) return st;
    double maxres = 0.0;
    for (int i = 0; i < k; ++i) maxres = std::max(maxres, resf[i]);
    inf.maxres = maxres;
    inf.converged = (done && maxres <= opts->tol) ? 1 : 0;
    if (done && !inf.converged) inf.exit_rule = 0;
    inf.spmm_blocks = c->spmm_blocks - spmm0;
    inf.p_final = p;
    inf.d_final = c->d;
    inf.locked = nc;
    for (int i = 0; i < k; ++i) { eigval_host[i] = c->sign * rf[i]; res_host[i] = resf[i]; }
    if (info) *info = inf;
    return ARR_OK;
}

// ---------------------------------------------------------------- column-partitioned mode
// (eig_init_colsplit; Survey §8f-3).  MPM filters every column independently
// (P:552-566), so with A replicated the filter of a column slice needs no
// communication at all; the ARR projection (Alg. ARR) needs the whole
// block and runs on a row-partitioned context after an all-to-all transpose.
namespace {
arr_status cs_solve(arr_ctx *c, double *X, int64_t ldx, const arr_solve_opts *opts, double *eigval_host,
                    double *res_host, arr_solve_info *info) {
    ColSplit &S = *c->cs;
    arr_ctx *cc = S.col, *cr = S.row;
    if (opts->adapt || opts->gn || opts->inner || opts->exits)
        return fail(c, ARR_EINVAL, "column split: only the fixed-parameter solve (no adapt / gn / inner / exits)");
    const int w = c->w, k = c->k;
    const int m = m_of(cr, cr->p);
    std::vector<double> ritz(m), res(k), r0(w);
    arr_solve_info inf{};
    double a = 0.0;
    arr_status st = eig_gershgorin_lower(cc, &a);  // the full A on every rank: the same bound
    if (st != ARR_OK) return st;
    if ((st = comm_transpose(c, S, 0, X, ldx, S.Xrow, S.ldrow)) != ARR_OK) return st;
    if ((st = arr_core(cr, 0, S.Xrow, S.ldrow, nullptr, 0, r0.data(), nullptr)) != ARR_OK) return st;
    double b = r0[w - 1], mu1 = r0[0];
    if (!(a < b)) a = b - 1e-8 * (fabs(b) + 1.0);
    const int64_t spmm0 = cc->spmm_blocks + cr->spmm_blocks;
    bool done = false, mono = false;
    double prev_maxres = 0.0;
    int32_t rank = 0;
    for (int outer = 1; outer <= opts->maxit; ++outer) {
        if ((st = eig_set_interval(cc, a, b)) != ARR_OK) return st;
        const double ccen = 0.5 * (a + b), e = 0.5 * (b - a);
        const double amp = fabs(cc->filter_kind == 1 ? psi_eval(cc->coef, (mu1 - ccen) / e) : chebT(cc->d, (mu1 - ccen) / e));
        const int s = sweeps_rule(amp, opts->s_max, opts->range_digits);
        CUDA_TRY(cudaMemsetAsync(cc->dinfo + INFO_BAD, 0, sizeof(int), cc->stream));
        for (int q = 0; q < s; ++q)
            if ((st = filter_core(cc, X, ldx, 1, nullptr)) != ARR_OK) return st;  // local: no exchange
        inf.sweeps += s;
        if ((st = comm_transpose(c, S, 0, X, ldx, S.Xrow, S.ldrow)) != ARR_OK) return st;
        if ((st = arr_core(cr, cr->p, S.Xrow, S.ldrow, S.Xrow, S.ldrow, ritz.data(), &rank)) != ARR_OK) return st;
        CUDA_TRY(cudaMemcpyAsync(cc->h_istage + 32, cc->dinfo + INFO_BAD, sizeof(int), cudaMemcpyDeviceToHost, cc->stream));
        if ((st = residuals_core(cr, S.Xrow, S.ldrow, ritz.data(), k, res.data())) != ARR_OK) return st;
        if ((st = comm_transpose(c, S, 1, S.Xrow, S.ldrow, X, ldx)) != ARR_OK) return st;  // Ritz vectors back
        // the flag is a per-rank local value; every rank stops together on any rank's flag
        c->h_stage[0] = cc->h_istage[32] ? 1.0 : 0.0;
        CUDA_TRY(cudaMemcpyAsync(cr->vecw, c->h_stage, sizeof(double), cudaMemcpyHostToDevice, c->stream));
        ST_TRY(comm_allreduce(cr, cr->vecw, 1, 2));
        CUDA_TRY(cudaMemcpyAsync(c->h_stage, cr->vecw, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (c->h_stage[0] != 0.0) return fail(c, ARR_ENUMERIC, "zero or non-finite column norm after filtering");
        double maxres = 0.0;
        for (int i = 0; i < k; ++i) maxres = std::max(maxres, res[i]);
        inf.outer = outer;
        inf.maxres = maxres;
        inf.last_rank = rank;
        inf.a = a; inf.b = b;
        if (maxres <= opts->tol) { done = true; inf.exit_rule = 1; break; }
        mono = mono || (outer > 1 && maxres > 10.0 * prev_maxres);  // R3, as eig_solve
        prev_maxres = maxres;
        const double bn = ritz[std::min(w, m - 1)];
        b = mono ? std::max(b, bn) : bn;
        mu1 = ritz[0];
        if (!(a < b)) a = b - 1e-8 * (fabs(b) + 1.0);
    }
    inf.p_final = cr->p;
    inf.d_final = cc->d;
    inf.converged = done ? 1 : 0;
    inf.spmm_blocks = cc->spmm_blocks + cr->spmm_blocks - spmm0;
    for (int i = 0; i < k; ++i) { eigval_host[i] = cr->sign * ritz[i]; res_host[i] = res[i]; }
    if (info) *info = inf;
    return ARR_OK;
}

void cs_release(arr_ctx *c) {
    ColSplit *S = c->cs;
    if (!S) return;
    cudaStreamSynchronize(c->stream);
    if (S->col) eig_destroy(S->col);
    if (S->row) eig_destroy(S->row);
    if (S->sendbuf) cudaFree(S->sendbuf);
    if (S->recvbuf) cudaFree(S->recvbuf);
    if (S->Xrow) cudaFree(S->Xrow);
    delete S;
    c->cs = nullptr;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

arr_status eig_init_colsplit(arr_ctx **out, const arr_csr *A_full, int32_t k, int32_t w, int32_t p, int32_t d,
                             const arr_csr *A_rows, const arr_dist *rows, const int64_t *row_begins,
                             const int64_t *col_begins, arr_comm *comm, void *stream) {
    if (!out || !A_full || !A_rows || !rows || !row_begins || !col_begins || !comm) return ARR_EINVAL;
    *out = nullptr;
    int32_t R = 0, G = 1;
    if (comm_rank_size(comm, &R, &G) != ARR_OK) return ARR_EINVAL;
    const int64_t n = A_full->n;
    if (row_begins[0] != 0 || row_begins[G] != n || col_begins[0] != 0 || col_begins[G] != w) return ARR_EINVAL;
    for (int q = 0; q < G; ++q)
        if (row_begins[q + 1] < row_begins[q] || col_begins[q + 1] <= col_begins[q]) return ARR_EINVAL;
    if (rows->row_begin != row_begins[R] || A_rows->n != row_begins[R + 1] - row_begins[R] || rows->n_global != n)
        return ARR_EINVAL;
    const int32_t wr = (int32_t)(col_begins[R + 1] - col_begins[R]);
    arr_ctx *c = new (std::nothrow) arr_ctx();
    if (!c) return ARR_ENOMEM;
    c->k = k; c->w = w; c->p = p; c->d = d;
    c->stream = (cudaStream_t)stream;
    c->poisoned = ARR_OK;
    c->comm = comm;
    c->nranks = G;
    c->sign = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
    ColSplit *S = new (std::nothrow) ColSplit();
    if (!S) { delete c; return ARR_ENOMEM; }
    c->cs = S;
    S->rb.assign(row_begins, row_begins + G + 1);
    S->cb.assign(col_begins, col_begins + G + 1);
    arr_status st = eig_init_w(&S->col, A_full, wr, wr, 0, d, stream);  // the filter of this rank's columns
    if (st == ARR_OK) st = eig_init_dist(&S->row, A_rows, k, w, p, d, rows, comm, stream);  // the ARR projection
    const int64_t nrow_blk = A_rows->n + rows->n_ghost;
    S->ldrow = ((int64_t)w + 1) & ~int64_t(1);
    const int64_t nr = row_begins[R + 1] - row_begins[R];
    S->buf_elems = (size_t)std::max<int64_t>(n * (((int64_t)wr + 1) & ~int64_t(1)), nr * ((int64_t)w + 2 * G));
    if (st == ARR_OK && (cudaMalloc(&S->Xrow, sizeof(double) * (size_t)nrow_blk * S->ldrow) != cudaSuccess ||
                         cudaMalloc(&S->sendbuf, sizeof(double) * S->buf_elems) != cudaSuccess ||
                         cudaMalloc(&S->recvbuf, sizeof(double) * S->buf_elems) != cudaSuccess ||
                         cudaMallocHost(&c->h_stage, sizeof(double) * 64) != cudaSuccess)) {
        cudaGetLastError();
        st = ARR_ENOMEM;
    }
    if (st != ARR_OK) {
        cs_release(c);
        if (c->h_stage) cudaFreeHost(c->h_stage);
        delete c;
        return st;
    }
    c->ws_bytes = S->col->ws_bytes + S->row->ws_bytes + sizeof(double) * ((size_t)nrow_blk * S->ldrow + 2 * S->buf_elems);
    if (!getenv("ARRABIT_COLSPLIT_ROWSPMM")) {  // the ARR's SpMMs in the column layout (default)
        S->row->cs_link = S;
        S->row->cs_outer = c;
    }
    *out = c;
    return ARR_OK;
}

arr_status eig_init(arr_ctx **out, const arr_csr *A, int32_t k, int32_t p, int32_t d, void *stream) {
    return eig_init_w(out, A, k, k, p, d, stream);
}

arr_status eig_init_dist(arr_ctx **out, const arr_csr *A, int32_t k, int32_t w_in, int32_t p, int32_t d,
                         const arr_dist *dist, arr_comm *comm, void *stream) {
    if (!out || !A) return ARR_EINVAL;
    *out = nullptr;
    if (A->n < 1 || A->n >= (int64_t(1) << 31) || A->nnz < 0 || !A->row_ptr || (A->nnz > 0 && (!A->col_idx || !A->val)))
        return ARR_EINVAL;
    int32_t crank = 0, csize = 1;
    if (comm && comm_rank_size(comm, &crank, &csize) != ARR_OK) return ARR_EINVAL;
    const bool multi = csize > 1;
    if (multi && !dist) return ARR_EINVAL;
    const int64_t n_global = multi ? dist->n_global : A->n;
    if (multi && (dist->n_ghost < 0 || A->n + dist->n_ghost >= (int64_t(1) << 31) || dist->row_begin < 0 ||
                  dist->row_begin + A->n > n_global))
        return ARR_EINVAL;
    if (k < 1 || w_in < k || p < 0 || p > ARR_MAX_P || d < 1 || (int64_t)(p + 1) * w_in >= n_global || w_in > ARR_MAX_W)
        return ARR_EINVAL;
    arr_ctx *c = new (std::nothrow) arr_ctx();
    if (!c) return ARR_ENOMEM;
    c->A = *A;
    c->k = k; c->w = w_in; c->p = p; c->d = d;
    c->stream = (cudaStream_t)stream;
    c->poisoned = ARR_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (c->num_sms <= 0) c->num_sms = 148;
    const int64_t n = A->n + (multi ? dist->n_ghost : 0), w = w_in, m = (int64_t)(p + 1) * w_in;
    const int64_t lq = ld_up(m), lt = ld_up(w);
    const int64_t mm = std::max<int64_t>(m, ARR_MAX_W);
    c->part_elems = (size_t)std::max<int64_t>(16 * m * w, 4096 * mm);
    struct Alloc { void **p; size_t bytes; };
    // Lean context (no scratch block T; Section "Memory" of DESIGN.md): when T and
    // the basis do not fit next to the caller's blocks, or on request (ARRABIT_LEAN)
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t need = sizeof(double) * (size_t)n * (size_t)(lt + lq) + ((size_t)1 << 30);
    const bool lean = p >= 1 && (getenv("ARRABIT_LEAN") != nullptr || need > free_b);
    std::vector<Alloc> al = {
        {(void **)&c->T, lean ? 0 : sizeof(double) * (size_t)n * lt},
        {(void **)&c->Q, sizeof(double) * (size_t)n * lq},
        {(void **)&c->part, sizeof(double) * c->part_elems},
        {(void **)&c->small, sizeof(double) * 4 * (size_t)m * m},
        {(void **)&c->evals, sizeof(double) * (size_t)m},
        {(void **)&c->vecw, sizeof(double) * 3 * (size_t)mm},
        {(void **)&c->dinfo, sizeof(int) * 64},
        {(void **)&c->sched, sizeof(unsigned long long) * 2},
        {(void **)&c->omega, sizeof(double) * (size_t)w * kOmegaCols},
        {(void **)&c->racc, sizeof(double) * 2 * (size_t)w * w},
        {(void **)&c->lazy, sizeof(double) * 2 * (ARR_MAX_W + 2)},
    };
    size_t total = 0;
    for (auto &x : al) {
        if (x.bytes == 0) { *x.p = nullptr; continue; }
        if (dev_alloc(x.p, x.bytes, c->stream) != cudaSuccess) {
            cudaGetLastError();
            eig_destroy(c);
            return ARR_ENOMEM;
        }
        total += x.bytes;
    }
    cudaMemsetAsync(c->dinfo, 0, sizeof(int) * 64, c->stream);
    cudaMemsetAsync(c->sched, 0, sizeof(unsigned long long) * 2, c->stream);
    {
        // the fixed sketch block of the re-orthogonality check: seeded N(0,1) (64-bit LCG + Box-Muller)
        std::vector<double> om((size_t)w * kOmegaCols);
        uint64_t st = 0x9E3779B97F4A7C15ull;
        auto u01 = [&]() { st = st * 6364136223846793005ull + 1442695040888963407ull; return ((st >> 11) + 0.5) * 0x1.0p-53; };
        for (size_t i = 0; i < om.size(); i += 2) {
            const double r = sqrt(-2.0 * log(u01())), t = 6.283185307179586 * u01();
            om[i] = r * cos(t);
            if (i + 1 < om.size()) om[i + 1] = r * sin(t);
        }
        if (cudaMemcpyAsync(c->omega, om.data(), sizeof(double) * om.size(), cudaMemcpyHostToDevice, c->stream) !=
                cudaSuccess ||
            cudaStreamSynchronize(c->stream) != cudaSuccess) {
            cudaGetLastError();
            eig_destroy(c);
            return ARR_ECUDA;
        }
    }
    if (solver_acquire(&c->solver) != CUSOLVER_STATUS_SUCCESS) { c->solver = nullptr; eig_destroy(c); return ARR_ECUSOLVER; }
    cusolverDnSetStream(c->solver, c->stream);
    int lwork = 0;
    if (cusolverDnDsyevd_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)m, c->small,
                                    (int)m, c->evals, &lwork) != CUSOLVER_STATUS_SUCCESS) {
        eig_destroy(c);
        return ARR_ECUSOLVER;
    }
    int lwork_w = 0;
    cusolverDnDsyevd_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, (int)w, c->small, (int)w,
                                c->evals, &lwork_w);
    int lwork_p = 0;
    cusolverDnDpotrf_bufferSize(c->solver, CUBLAS_FILL_MODE_UPPER, (int)w, c->small, (int)w, &lwork_p);
    int lwork_i = 0;
    cusolverDnDpotri_bufferSize(c->solver, CUBLAS_FILL_MODE_LOWER, (int)w, c->small, (int)w, &lwork_i);
    c->solver_lwork = std::max(std::max(std::max(lwork, lwork_w), lwork_p), lwork_i);
    size_t tdb = 0, thb = 0;
    if (cusolverDnXtrtri_bufferSize(c->solver, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, w, CUDA_R_64F, c->small, w,
                                    &tdb, &thb) != CUSOLVER_STATUS_SUCCESS) {
        eig_destroy(c);
        return ARR_ECUSOLVER;
    }
    c->trtri_dbytes = std::max<size_t>(tdb, 16);
    c->trtri_hwork.resize(std::max<size_t>(thb, 16));
    if (dev_alloc(&c->trtri_dwork, c->trtri_dbytes, c->stream) != cudaSuccess) {
        cudaGetLastError();
        eig_destroy(c);
        return ARR_ENOMEM;
    }
    c->orth_mode = getenv("ARRABIT_ORTH_SVQB") ? 1 : 0;
    c->sign = 1;
    c->tile_rows = 32;  // measured best on B200 for cfg2 (with the L2 prefetch) and cfg3 natural order
    if (const char *tr = getenv("ARRABIT_TILE")) c->tile_rows = std::min(64, std::max(1, atoi(tr)));
    c->col_split = 1;
    if (const char *cs = getenv("ARRABIT_SPLIT")) c->col_split = std::min(4, std::max(1, atoi(cs)));
    if (dev_alloc((void **)&c->solver_work, sizeof(double) * (size_t)c->solver_lwork, c->stream) != cudaSuccess) {
        cudaGetLastError();
        eig_destroy(c);
        return ARR_ENOMEM;
    }
    total += sizeof(double) * (size_t)c->solver_lwork;
    if (cudaMallocHost(&c->h_stage, sizeof(double) * (size_t)(mm + 64)) != cudaSuccess ||
        cudaMallocHost(&c->h_istage, sizeof(int) * 64) != cudaSuccess) {
        cudaGetLastError();
        eig_destroy(c);
        return ARR_ENOMEM;
    }
    c->ws_bytes = total;
    if (multi) {
        if (comm_setup_plan(c, dist, comm) != ARR_OK) {
            const arr_status e = c->poisoned != ARR_OK ? c->poisoned : ARR_EINVAL;
            fprintf(stderr, "eig_init_dist: %s\n", c->err.c_str());
            eig_destroy(c);
            return e;
        }
    }
    launch_rowlen_max(c, c->dinfo + 63);
    if (cudaMemcpyAsync(c->h_istage, c->dinfo + 63, sizeof(int), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess) {
        cudaGetLastError();
        eig_destroy(c);
        return ARR_ECUDA;
    }
    c->max_row_nnz = c->h_istage[0];
    if (multi) {  // one chunk size on every rank (the per-row arithmetic does not depend on it)
        c->h_stage[0] = (double)c->max_row_nnz;
        if (cudaMemcpyAsync(c->vecw, c->h_stage, sizeof(double), cudaMemcpyHostToDevice, c->stream) != cudaSuccess ||
            comm_allreduce(c, c->vecw, 1, 2) != ARR_OK ||
            cudaMemcpyAsync(c->h_stage, c->vecw, sizeof(double), cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
            cudaStreamSynchronize(c->stream) != cudaSuccess) {
            eig_destroy(c);
            return ARR_ENCCL;
        }
        c->max_row_nnz = (int)c->h_stage[0];
    }
    *out = c;
    return ARR_OK;
}

arr_status eig_init_w(arr_ctx **out, const arr_csr *A, int32_t k, int32_t w_in, int32_t p, int32_t d, void *stream) {
    return eig_init_dist(out, A, k, w_in, p, d, nullptr, nullptr, stream);
}

arr_status eig_destroy(arr_ctx *c) {
    if (!c) return ARR_EINVAL;
    if (c->cs) {
        cs_release(c);
        if (c->h_stage) cudaFreeHost(c->h_stage);
        delete c;
        return ARR_OK;
    }
    cudaStreamSynchronize(c->stream);
    for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
    if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
    stencil_release(c);
    void *ptrs[] = {c->T, c->Q, c->part, c->small, c->evals, c->vecw, c->dinfo, c->sched, c->solver_work,
                    c->trtri_dwork, c->omega, c->lazy};
    for (void *p : ptrs)
        dev_free(p, c->stream);
    cudaStreamSynchronize(c->stream);
    if (c->h_stage) cudaFreeHost(c->h_stage);
    if (c->h_istage) cudaFreeHost(c->h_istage);
    if (c->solver) solver_release(c->solver);
    comm_free_plan(c);
    delete c;
    return ARR_OK;
}

const char *eig_last_error(const arr_ctx *c) { return c ? c->err.c_str() : "null context"; }
size_t eig_workspace_bytes(const arr_ctx *c) { return c ? c->ws_bytes : 0; }
uint64_t eig_launch_count(const arr_ctx *c) {
    if (c && c->cs) return c->launches + c->cs->col->launches + c->cs->row->launches;
    return c ? c->launches : 0;
}

arr_status eig_gershgorin_lower(arr_ctx *c, double *a_out) {
    GUARD(c);
    if (c->cs) return eig_gershgorin_lower(c->cs->col, a_out);
    if (!a_out) return fail(c, ARR_EINVAL, "a_out is NULL");
    int nb = 0;
    launch_gershgorin(c, c->part, &nb);
    launch_min_finalize(c, c->part, nb, NORM_buf(c));
    CHECK_LAUNCH();
    ST_TRY(comm_allreduce(c, NORM_buf(c), 1, 1));
    CUDA_TRY(cudaMemcpyAsync(c->h_stage, NORM_buf(c), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    *a_out = c->h_stage[0];
    return ARR_OK;
}

arr_status eig_set_interval(arr_ctx *c, double a, double b) {
    GUARD(c);
    if (c->cs) ST_TRY(eig_set_interval(c->cs->col, a, b));
    if (!(a < b) || !isfinite(a) || !isfinite(b)) return fail(c, ARR_EINVAL, "interval needs finite a < b");
    c->a = a; c->b = b; c->have_interval = true;
    return ARR_OK;
}

arr_status eig_set_schedule(arr_ctx *c, const int64_t *tile_row0, const int32_t *tile_len, int64_t ntiles) {
    GUARD(c);
    if (c->cs) return eig_set_schedule(c->cs->col, tile_row0, tile_len, ntiles);
    if (is_dist(c)) return fail(c, ARR_EINVAL, "schedule: not supported on a distributed context");
    if (!tile_row0) {
        c->tile_row0 = nullptr; c->tile_len = nullptr; c->ntiles = 0;
        return ARR_OK;
    }
    if (!tile_len || ntiles < 1) return fail(c, ARR_EINVAL, "schedule: null lengths or no tiles");
    int *marks = reinterpret_cast<int *>(c->T ? c->T : c->Q);  // a scratch block holds >= n ints
    launch_schedule_check(c, tile_row0, tile_len, ntiles, marks, c->dinfo + INFO_BAD);
    CHECK_LAUNCH();
    CUDA_TRY(cudaMemcpyAsync(c->h_istage, c->dinfo + INFO_BAD, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->h_istage[0]) return fail(c, ARR_EINVAL, "schedule does not cover every row exactly once with tiles of 1..64 rows");
    c->tile_row0 = tile_row0; c->tile_len = tile_len; c->ntiles = ntiles;
    return ARR_OK;
}

arr_status eig_set_stencil(arr_ctx *c, int64_t nx, int64_t ny, int64_t nz) {
    GUARD(c);
    if (c->cs) return eig_set_stencil(c->cs->col, nx, ny, nz);  // the column context has the whole A
    int gz_lo = 0, gz_hi = 0;
    if (is_dist(c) && (nx || ny || nz)) {
        // z-slab of a row partition: (nx, ny, nz) is this rank's slab of whole grid planes; the
        // ghost rows must be the whole plane below (from lower ranks) and / or above
        const DistPlan &P = c->plan;
        int32_t my_rank = 0, nr = 1;
        comm_rank_size(c->comm, &my_rank, &nr);
        int64_t lo = 0, hi = 0;
        bool ordered = true;  // every lower-rank peer's rows before every higher-rank peer's
        for (size_t q = 0; q < P.peer.size(); ++q) {
            const int64_t cnt = P.recv_off[q + 1] - P.recv_off[q];
            if (P.peer[q] < my_rank) { lo += cnt; ordered = ordered && hi == 0; }
            else hi += cnt;
        }
        const int64_t nxy = nx * ny;
        if (nx < 1 || ny < 1 || nz < 1 || !ordered || (lo != 0 && lo != nxy) || (hi != 0 && hi != nxy) ||
            lo + hi != P.n_ghost)
            return fail(c, ARR_EINVAL, "eig_set_stencil on a row partition: the rank's rows must be a z-slab of whole "
                                       "grid planes whose ghost rows are the neighbouring planes");
        gz_lo = lo ? 1 : 0;
        gz_hi = hi ? 1 : 0;
    }
    const arr_status st = stencil_setup(c, nx, ny, nz, gz_lo, gz_hi);
    if (st == ARR_OK && is_dist(c) && c->st.on) {
        // are the plan's boundary tiles exactly the slab's end planes?
        const DistPlan &P = c->plan;
        const int64_t nxy = nx * ny, nown = c->A.n;
        std::vector<int64_t> r0((size_t)P.n_bnd_tiles);
        std::vector<int32_t> ln((size_t)P.n_bnd_tiles);
        if (P.n_bnd_tiles > 0) {
            CUDA_TRY(cudaMemcpyAsync(r0.data(), P.bnd_row0, sizeof(int64_t) * r0.size(), cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaMemcpyAsync(ln.data(), P.bnd_len, sizeof(int32_t) * ln.size(), cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaStreamSynchronize(c->stream));
        }
        int64_t total = 0;
        bool inside = true;
        for (size_t t = 0; t < r0.size(); ++t) {
            const int64_t a0 = r0[t], a1 = r0[t] + ln[t];
            const bool in_lo = gz_lo && a1 <= nxy, in_hi = gz_hi && a0 >= nown - nxy;
            inside = inside && (in_lo || in_hi);
            total += ln[t];
        }
        c->st.bnd_is_ends = inside && nz >= 2 && total == (int64_t)(gz_lo + gz_hi) * nxy;
    }
    if (st == ARR_EINVAL)
        return fail(c, st, "eig_set_stencil: n != nx*ny*nz, or a row of A is unsorted / has a column outside the "
                           "3x3x3 neighbourhood of its grid point");
    if (st != ARR_OK) return fail(c, st, "eig_set_stencil failed");
    return ARR_OK;
}

int32_t eig_stencil_active(const arr_ctx *c) {
    if (c && c->cs) return eig_stencil_active(c->cs->col);
    return c && c->st.on ? c->st.K : 0;
}

int32_t eig_stencil_abytes(const arr_ctx *c) {
    if (c && c->cs) return eig_stencil_abytes(c->cs->col);
    if (!c || !c->st.on) return -1;
    return c->st.vmode == 0 ? 8 * c->st.K : (c->st.vmode == 1 ? 8 : 0);
}
const char *eig_last_spmm_kernel(const arr_ctx *c) {
    if (c && c->cs) return eig_last_spmm_kernel(c->cs->col);
    return c && c->last_kernel ? c->last_kernel : "";
}

arr_status eig_set_degree(arr_ctx *c, int32_t d) {
    GUARD(c);
    if (c->cs) { ST_TRY(eig_set_degree(c->cs->col, d)); ST_TRY(eig_set_degree(c->cs->row, d)); c->d = d; return ARR_OK; }
    if (d < 1) return fail(c, ARR_EINVAL, "degree must be >= 1");
    c->d = d;
    if (c->filter_kind == 1) c->coef = interp_coef(d);
    return ARR_OK;
}

arr_status eig_set_mode(arr_ctx *c, int32_t smallest) {
    GUARD(c);
    if (c->cs) { ST_TRY(eig_set_mode(c->cs->col, smallest)); ST_TRY(eig_set_mode(c->cs->row, smallest)); }
    c->sign = smallest ? -1 : 1;
    c->have_interval = false;  // an interval of A is not one of -A
    return ARR_OK;
}

arr_status eig_set_filter(arr_ctx *c, int32_t kind) {
    GUARD(c);
    if (c->cs) return eig_set_filter(c->cs->col, kind);
    if (kind != 0 && kind != 1) return fail(c, ARR_EINVAL, "filter kind must be 0 (T_d) or 1 (psi_d)");
    if (kind == 1 && !c->T && c->p < 1)
        return fail(c, ARR_EINVAL, "the interpolant filter needs two scratch blocks (p >= 1 in a lean context)");
    c->filter_kind = kind;
    c->coef = kind == 1 ? interp_coef(c->d) : std::vector<double>();
    return ARR_OK;
}

arr_status filter_step(arr_ctx *c, double *X, int64_t ldx, int32_t normalize, double *colnorm_dev) {
    GUARD_KEEP(c);
    if (normalize < 0 || normalize > 2) return fail(c, ARR_EINVAL, "filter_step: normalize must be 0, 1 or 2");
    Nvtx nvtx_("arrabit::filter_step");
    if (c->cs) return filter_step(c->cs->col, X, ldx, normalize, colnorm_dev);  // this rank's columns: no exchange
    if (!c->have_interval) return fail(c, ARR_EINVAL, "eig_set_interval not called");
    if (!block_ok(X, ldx, c->w)) return fail(c, ARR_EINVAL, "bad block X / ldx");
    CUDA_TRY(cudaMemsetAsync(c->dinfo + INFO_BAD, 0, sizeof(int), c->stream));
    arr_status st = filter_core(c, X, ldx, normalize, colnorm_dev);
    if (st != ARR_OK) return st;
    if (normalize) {
        CUDA_TRY(cudaMemcpyAsync(c->h_istage, c->dinfo + INFO_BAD, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        t_resolve(c);
        if (c->h_istage[0]) return fail(c, ARR_ENUMERIC, "zero or non-finite column norm after filtering");
    }
    return ARR_OK;
}

arr_status eig_set_timing(arr_ctx *c, int32_t on) {
    GUARD(c);
    if (c->cs) { ST_TRY(eig_set_timing(c->cs->col, on)); ST_TRY(eig_set_timing(c->cs->row, on)); }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    c->pending.clear();
    c->ev_next = 0;
    c->timing = on != 0;
    for (int i = 0; i < kPhasesAll; ++i) { c->phase_ms[i] = 0.0; c->phase_cnt[i] = 0; c->phase_work[i] = 0.0; }
    return ARR_OK;
}

arr_status eig_phase_times(arr_ctx *c, double *ms, int64_t *counts) {
    GUARD(c);
    if (!ms || !counts) return fail(c, ARR_EINVAL, "null output");
    if (c->cs) {  // filter degrees from the column context, the ARR / residual phases from the row context
        double m2[kPhases];
        int64_t c2[kPhases];
        ST_TRY(eig_phase_times(c->cs->col, ms, counts));
        ST_TRY(eig_phase_times(c->cs->row, m2, c2));
        for (int i = 1; i < kPhases; ++i) { ms[i] = m2[i]; counts[i] = c2[i]; }
        return ARR_OK;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    t_resolve(c);
    for (int i = 0; i < kPhases; ++i) { ms[i] = c->phase_ms[i]; counts[i] = c->phase_cnt[i]; }
    return ARR_OK;
}

arr_status eig_kernel_times(arr_ctx *c, double *ms, double *flops, int64_t *launches) {
    GUARD(c);
    if (!ms || !flops || !launches) return fail(c, ARR_EINVAL, "null output");
    arr_ctx *t = c->cs ? c->cs->row : c;  // the column split's ARR runs on its row context
    CUDA_TRY(cudaStreamSynchronize(t->stream));
    t_resolve(t);
    for (int i = 0; i < 2; ++i) {
        ms[i] = t->phase_ms[6 + i];
        flops[i] = t->phase_work[6 + i];
        launches[i] = t->phase_cnt[6 + i];
    }
    return ARR_OK;
}

arr_status spmm(arr_ctx *c, double alpha, double shift, const double *X, int64_t ldx, double *Y, int64_t ldy,
                int32_t ncols) {
    GUARD(c);
    if (c->cs) return spmm(c->cs->col, alpha, shift, X, ldx, Y, ldy, ncols);  // whole A, this rank's columns
    if (!block_ok(X, ldx, ncols) || !block_ok(Y, ldy, ncols) || ncols > ARR_MAX_W)
        return fail(c, ARR_EINVAL, "bad block / ncols");
    SpmmArgs s{};
    s.row_ptr = c->A.row_ptr; s.col = c->A.col_idx; s.val = c->A.val;
    s.n = c->A.n; s.w = ncols;
    s.Yin = X; s.ld_in = ldx;
    s.alpha = alpha; s.shift = shift;
    s.Yout = Y; s.ld_out = ldy;
    arr_status st;
    const int g = spmm_x(c, s, &st, /*op=*/false);  // A itself (not the solver's operator sign*A)
    if (st != ARR_OK) return st;
    if (g < 0) return fail(c, ARR_EINVAL, "unsupported width");
    CHECK_LAUNCH();
    return ARR_OK;
}

arr_status gram(arr_ctx *c, const double *X, int64_t ldx, int32_t m1, const double *Y, int64_t ldy, int32_t m2,
                double *G, int64_t ldg) {
    GUARD(c);
    if (c->cs) return fail(c, ARR_EINVAL, "gram: not available on a column-split context");
    if (!block_ok(X, ldx, m1) || !block_ok(Y, ldy, m2) || !G || ldg < m2) return fail(c, ARR_EINVAL, "bad gram args");
    if ((size_t)m1 * (size_t)m2 > c->part_elems)
        return fail(c, ARR_EINVAL, "gram: m1 * m2 exceeds the context's partial-sum buffer (m1 * m2 <= " +
                                       std::to_string(c->part_elems) + ")");
    ST_TRY(gram_x(c, X, ldx, m1, Y, ldy, m2, G, ldg));
    CHECK_LAUNCH();
    return ARR_OK;
}

arr_status gemm(arr_ctx *c, double alpha, const double *X, int64_t ldx, int32_t m1, const double *B, int64_t ldb,
                int32_t m2, double beta, const double *Cin, int64_t ldc, double *Out, int64_t ldo) {
    GUARD(c);
    if (c->cs) return fail(c, ARR_EINVAL, "gemm: not available on a column-split context");
    if (!block_ok(X, ldx, m1) || !B || ldb < m2 || !block_ok(Out, ldo, m2) || (beta != 0.0 && !block_ok(Cin, ldc, m2)))
        return fail(c, ARR_EINVAL, "bad gemm args");
    if ((const void *)X == (const void *)Out) return fail(c, ARR_EINVAL, "gemm: X aliases Out");
    launch_gemm(c, alpha, X, ldx, m1, B, ldb, m2, beta, Cin, ldc, Out, ldo, c->A.n);
    CHECK_LAUNCH();
    return ARR_OK;
}

arr_status orthonormalize(arr_ctx *c, double *X, int64_t ldx, int32_t ncols, int32_t *rank) {
    GUARD(c);
    Nvtx nvtx_("arrabit::orthonormalize");
    if (c->cs) return fail(c, ARR_EINVAL, "orthonormalize: not available on a column-split context");
    if (!block_ok(X, ldx, ncols) || ncols > c->w) return fail(c, ARR_EINVAL, "bad block / ncols > w");
    // keep the input in the basis buffer: CholeskyQR3 X_copy -> X, SVQB fallback from the copy
    launch_copy_rows(c, X, ldx, c->Q, ldQ(c), c->A.n, ncols);
    bool ok = false;
    arr_status st;
    double *S = c->T ? c->T : c->Q + c->w;  // lean: the spare basis block (p >= 1)
    const int64_t ls = c->T ? ldT(c) : ldQ(c);
    if (c->orth_mode == 0 &&
        (st = cholqr3(c, c->Q, ldQ(c), X, ldx, ncols, c->dinfo + INFO_RANK0, &ok, S, ls)) != ARR_OK)
        return st;
    if (!ok && (st = svqb2(c, c->Q, ldQ(c), X, ldx, ncols, c->dinfo + INFO_RANK0, S, ls)) != ARR_OK) return st;
    CUDA_TRY(cudaMemcpyAsync(c->h_istage, c->dinfo, sizeof(int) * (INFO_RANK0 + 1), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->h_istage[INFO_SYEVD] != 0) return fail(c, ARR_ECUSOLVER, "syevd failed");
    if (rank) *rank = c->h_istage[INFO_RANK0];
    return ARR_OK;
}

arr_status arr_project_p(arr_ctx *c, int32_t p_use, const double *X, int64_t ldx, double *Y, int64_t ldy,
                         double *ritz_host, int32_t *rank) {
    GUARD(c);
    Nvtx nvtx_("arrabit::arr_project");
    if (c->cs) {  // column layout -> rows, the row context's ARR, Ritz vectors back to this rank's columns
        ColSplit &S = *c->cs;
        if (!block_ok(X, ldx, S.col->w) || (Y && !block_ok(Y, ldy, S.col->w)) || !ritz_host)
            return fail(c, ARR_EINVAL, "bad arr_project args (column slices)");
        ST_TRY(comm_transpose(c, S, 0, X, ldx, S.Xrow, S.ldrow));
        ST_TRY(arr_project_p(S.row, p_use, S.Xrow, S.ldrow, Y ? S.Xrow : nullptr, S.ldrow, ritz_host, rank));
        if (Y) ST_TRY(comm_transpose(c, S, 1, S.Xrow, S.ldrow, Y, ldy));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        return ARR_OK;
    }
    if (p_use < 0 || p_use > c->p) return fail(c, ARR_EINVAL, "p_use out of range");
    if (!block_ok(X, ldx, c->w) || (Y && !block_ok(Y, ldy, c->w)) || !ritz_host)
        return fail(c, ARR_EINVAL, "bad arr_project args");
    if (!c->T && p_use > 0 && (Y != X || ldy != ldx))
        return fail(c, ARR_EINVAL, "lean context (no scratch block): arr_project with p > 0 needs Y == X");
    arr_status st = arr_core(c, p_use, X, ldx, Y, ldy, ritz_host, rank);
    if (st == ARR_OK && c->sign < 0)
        for (int i = 0; i < (p_use + 1) * c->w; ++i) ritz_host[i] = -ritz_host[i];  // eigenvalues of A, ascending
    return st;
}

arr_status arr_project(arr_ctx *c, const double *X, int64_t ldx, double *Y, int64_t ldy, double *ritz_host,
                       int32_t *rank) {
    GUARD(c);
    return arr_project_p(c, c->p, X, ldx, Y, ldy, ritz_host, rank);
}

arr_status residuals(arr_ctx *c, const double *Y, int64_t ldy, const double *mu_host, int32_t ncols,
                     double *res_host) {
    GUARD(c);
    Nvtx nvtx_("arrabit::residuals");
    if (c->cs) {  // the block's columns gathered as rows, then the row context's residual pass
        ColSplit &S = *c->cs;
        if (ncols > c->w || !block_ok(Y, ldy, S.col->w)) return fail(c, ARR_EINVAL, "column split: ncols > w or bad Y");
        ST_TRY(comm_transpose(c, S, 0, Y, ldy, S.Xrow, S.ldrow));
        return residuals(S.row, S.Xrow, S.ldrow, mu_host, ncols, res_host);
    }
    if (!block_ok(Y, ldy, ncols) || ncols > std::max(m_of(c, c->p), ARR_MAX_W) || !mu_host || !res_host)
        return fail(c, ARR_EINVAL, "bad residual args");
    if (c->sign > 0) return residuals_core(c, Y, ldy, mu_host, ncols, res_host);
    std::vector<double> mu(mu_host, mu_host + ncols);  // eigenvalues of A -> of the operator -A
    for (auto &x : mu) x = -x;
    return residuals_core(c, Y, ldy, mu.data(), ncols, res_host);
}

arr_status eig_solve(arr_ctx *c, double *X, int64_t ldx, const arr_solve_opts *opts, double *eigval_host,
                     double *res_host, arr_solve_info *info) {
    GUARD(c);
    Nvtx nvtx_("arrabit::eig_solve");
    if (c->cs) {
        if (!block_ok(X, ldx, c->cs->col->w) || !opts || !eigval_host || !res_host) return fail(c, ARR_EINVAL, "bad solve args");
        return cs_solve(c, X, ldx, opts, eigval_host, res_host, info);
    }
    if (!block_ok(X, ldx, c->w) || !opts || !eigval_host || !res_host) return fail(c, ARR_EINVAL, "bad solve args");
    if (opts->gn && (c->p < 1 || (c->filter_kind == 1 && (c->T ? c->p < 1 : c->p < 2))))
        return fail(c, ARR_EINVAL, "GN inner solver: needs a spare basis block (p >= 1; p >= 2 with psi_d in a lean context)");
    if (opts->adapt & 4) {
        // continuation + deflation runs the fixed-p/d MPM sweeps of solve_deflate only
        if ((opts->adapt & 3) || opts->gn || opts->inner != 0 || opts->exits != 0)
            return fail(c, ARR_EINVAL, "adapt bit 4 (continuation + deflation) cannot be combined with adaptive p/d, "
                                       "GN, the rcond inner rule or the extra exit rules");
        return solve_deflate(c, X, ldx, opts, eigval_host, res_host, info);
    }
    const int w = c->w, k = c->k;
    const int m = m_of(c, c->p);
    std::vector<double> ritz(m), res(k);
    arr_solve_info inf{};
    double a = 0.0;
    arr_status st = eig_gershgorin_lower(c, &a);
    if (st != ARR_OK) return st;
    // b: smallest Ritz value of RR(A, X0)
    std::vector<double> r0(w);
    if ((st = arr_core(c, 0, X, ldx, nullptr, 0, r0.data(), nullptr)) != ARR_OK) return st;
    double b = r0[w - 1], mu1 = r0[0];
    if (!(a < b)) a = b - 1e-8 * (fabs(b) + 1.0);
    const int64_t spmm0 = c->spmm_blocks;
    bool done = false, mono = false;
    std::vector<double> best_hist;
    // adaptive augmentation depth and degree (Alg. Arrabit2, Eqs. block / hat-d / degree,
    // P:1418-1456), opt-in: p grows from 1 up to the context's p; d starts at 3 and is
    // re-chosen after every ARR, capped by the context's d (the paper's d_max)
    const int p_max = c->p, d_max = c->d;
    int p_cur = (opts->adapt & 1) ? std::min(1, p_max) : p_max;
    if ((opts->adapt & 2) && d_max > 3 && (st = eig_set_degree(c, 3)) != ARR_OK) return st;
    double best_res = INFINITY, best_muk = 0.0, best_muw = 0.0, maxresp = INFINITY;
    double prev_maxres = 0.0;
    int32_t rank = 0;
    for (int outer = 1; outer <= opts->maxit; ++outer) {
        if ((st = eig_set_interval(c, a, b)) != ARR_OK) return st;
        // sweeps between ARR steps: dynamic-range rule (R6)
        const double cc = 0.5 * (a + b), e = 0.5 * (b - a);
        const double amp = fabs(c->filter_kind == 1 ? psi_eval(c->coef, (mu1 - cc) / e) : chebT(c->d, (mu1 - cc) / e));
        int s = sweeps_rule(amp, opts->s_max, opts->range_digits);
        CUDA_TRY(cudaMemsetAsync(c->dinfo + INFO_BAD, 0, sizeof(int), c->stream));
        if (opts->inner == 1) {
            // the paper's inner stop: every maxit_2 = 5 sweeps, at most maxit_1 = 10
            // times, rc = rcond(X^T X); stop when rc <= tol or rc / rc_prev > 0.99 (rcond taken in the
            // 2-norm, lambda_min / lambda_max of the Gram: DESIGN.md R6)
            double rcp = -1.0;
            s = 0;
            for (int chk = 0; chk < 10; ++chk) {
                for (int q = 0; q < 5; ++q) {
                    st = opts->gn ? gn_step(c, X, ldx) : filter_core(c, X, ldx, 1, nullptr);
                    if (st != ARR_OK) return st;
                }
                s += 5;
                double rc = 0.0;
                if ((st = gram_rcond(c, X, ldx, &rc)) != ARR_OK) return st;
                if (rc <= opts->tol || (rcp > 0.0 && rc / rcp > 0.99)) break;
                rcp = rc;
            }
        } else {
            // MPM sweeps with the column normalisation folded lazily into the next
            // sweep (Survey §8a A2); the sweep before the ARR normalises explicitly
            static const bool lazy = [] { const char *e = getenv("ARRABIT_LAZY_NORM"); return !(e && atoi(e) == 0); }();
            for (int q = 0; q < s; ++q) {
                if (opts->gn) st = gn_step(c, X, ldx);             // GN inner solver
                else st = filter_core(c, X, ldx, (lazy && q + 1 < s) ? 2 : 1, nullptr);
                if (st != ARR_OK) return st;
            }
        }
        inf.sweeps += s;
        if ((st = arr_core(c, p_cur, X, ldx, X, ldx, ritz.data(), &rank)) != ARR_OK) return st;  // ARR
        CUDA_TRY(cudaMemcpyAsync(c->h_istage + 32, c->dinfo + INFO_BAD, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        if ((st = residuals_core(c, X, ldx, ritz.data(), k, res.data())) != ARR_OK) return st;  // Eq. resi
        if (c->h_istage[32]) return fail(c, ARR_ENUMERIC, "zero or non-finite column norm after filtering");
        double maxres = 0.0;
        for (int i = 0; i < k; ++i) maxres = std::max(maxres, res[i]);
        inf.outer = outer;
        inf.maxres = maxres;
        inf.last_rank = rank;
        inf.a = a; inf.b = b;
        log_outer(opts, outer, s, a, b, mu1, maxres, p_cur, c->d, 0, opts->tol, ritz[k - 1], ritz[w - 1]);
        if (maxres <= opts->tol) { done = true; inf.exit_rule = 1; break; }  // Eq. out-stop
        // the paper's extra stop rules, opt-in (R10)
        if (opts->exits & 1) {
            best_hist.push_back(maxres);
            const size_t h = best_hist.size();
            if (h >= 4 && !(best_hist[h - 1] < best_hist[h - 4] || best_hist[h - 2] < best_hist[h - 4] ||
                            best_hist[h - 3] < best_hist[h - 4])) {
                inf.exit_rule = 2;  // (ii): not reduced over three consecutive outer iterations
                break;
            }
        }
        if (opts->exits & 2) {
            int hsmall = 0;
            for (int i = 0; i < k; ++i) hsmall += res[i] < 0.1 * opts->tol;
            if (maxres < (1.0 + 9.0 * hsmall / k) * opts->tol) { inf.exit_rule = 3; break; }  // (iii)
        }
        // b = mu_{w+1}, an under-estimate of lambda_{k+q} (interlacing); once
        // the max residual has grown tenfold between two outer iterations, b only increases (R3)
        mono = mono || (outer > 1 && maxres > 10.0 * prev_maxres);
        prev_maxres = maxres;
        const double bn = ritz[std::min(w, m_of(c, p_cur) - 1)];
        b = mono ? std::max(b, bn) : bn;
        mu1 = ritz[0];
        if (!(a < b)) a = b - 1e-8 * (fabs(b) + 1.0);
        if (maxres < best_res) { best_res = maxres; best_muk = ritz[k - 1]; best_muw = ritz[w - 1]; }
        if ((opts->adapt & 1) && p_cur < p_max) {  // Eq. block: small decay and unimpressive progress
            const double decay = (ritz[w - 1] - a) / (ritz[k - 1] - a);
            if (decay > 0.95 && maxres / maxresp > 0.1) ++p_cur;
        }
        maxresp = maxres;
        if ((opts->adapt & 2) && d_max > 3) {  // Eqs. hat-d, degree: smallest d >= 3 separating mu*_{k+q} from mu*_k
            const double cc2 = 0.5 * (a + b), e2 = 0.5 * (b - a);
            int dn = d_max;
            for (int dd = 3; dd <= d_max; ++dd) {
                double rk, rw;
                if (c->filter_kind == 1) {
                    const std::vector<double> cf = interp_coef(dd);
                    rk = psi_eval(cf, (best_muk - cc2) / e2);
                    rw = psi_eval(cf, (best_muw - cc2) / e2);
                } else {
                    rk = chebT(dd, (best_muk - cc2) / e2);
                    rw = chebT(dd, (best_muw - cc2) / e2);
                }
                if (fabs(rw) < 0.9 * fabs(rk)) { dn = dd; break; }
            }
            if (dn != c->d && (st = eig_set_degree(c, dn)) != ARR_OK) return st;
        }
    }
    inf.p_final = p_cur;
    inf.d_final = c->d;
    if ((opts->adapt & 2) && c->d != d_max && (st = eig_set_degree(c, d_max)) != ARR_OK) return st;
    inf.converged = done ? 1 : 0;
    inf.spmm_blocks = c->spmm_blocks - spmm0;
    for (int i = 0; i < k; ++i) { eigval_host[i] = c->sign * ritz[i]; res_host[i] = res[i]; }
    if (info) *info = inf;
    return ARR_OK;
}

arr_status eig_solve_host(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx, const double *val,
                          int32_t k, int32_t w, int32_t p, int32_t d, const double *X0, const arr_solve_opts *opts,
                          double *eigval, double *res, double *evec, arr_solve_info *info, void *stream) {
    if (!row_ptr || !col_idx || !val || !X0 || !opts || !eigval || !res || n < 1 || k < 1 || w < k) return ARR_EINVAL;
    cudaStream_t s = (cudaStream_t)stream;
    int64_t *d_rp = nullptr;
    int32_t *d_ci = nullptr;
    double *d_val = nullptr, *d_X = nullptr;
    arr_ctx *c = nullptr;
    arr_status st = ARR_OK;
    const int64_t ldx = ld_up(w);
    auto cleanup = [&]() {
        if (c) eig_destroy(c);
        dev_free(d_rp, s); dev_free(d_ci, s); dev_free(d_val, s); dev_free(d_X, s);
        cudaStreamSynchronize(s);
    };
    if (dev_alloc((void **)&d_rp, sizeof(int64_t) * (n + 1), s) != cudaSuccess ||
        dev_alloc((void **)&d_ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1), s) != cudaSuccess ||
        dev_alloc((void **)&d_val, sizeof(double) * std::max<int64_t>(nnz, 1), s) != cudaSuccess ||
        dev_alloc((void **)&d_X, sizeof(double) * n * ldx, s) != cudaSuccess) {
        cudaGetLastError();
        cleanup();
        return ARR_ENOMEM;
    }
    if (cudaMemcpyAsync(d_rp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(d_ci, col_idx, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(d_val, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpy2DAsync(d_X, sizeof(double) * ldx, X0, sizeof(double) * w, sizeof(double) * w, n,
                          cudaMemcpyHostToDevice, s) != cudaSuccess) {
        cleanup();
        return ARR_ECUDA;
    }
    arr_csr A{n, nnz, d_rp, d_ci, d_val};
    st = eig_init_w(&c, &A, k, w, p, d, stream);
    if (st == ARR_OK)  // keep this call's footprint in the pool for the next call (dev_alloc)
        pool_keep_at_least((uint64_t)c->ws_bytes + sizeof(double) * (uint64_t)n * ldx +
                           (sizeof(int64_t) * (n + 1) + (sizeof(int32_t) + sizeof(double)) * (uint64_t)nnz));
    if (st == ARR_OK && (opts->grid[0] || opts->grid[1] || opts->grid[2]))
        st = eig_set_stencil(c, opts->grid[0], opts->grid[1], opts->grid[2]);
    if (st == ARR_OK) st = eig_solve(c, d_X, ldx, opts, eigval, res, info);
    if (st == ARR_OK && evec) {
        if (cudaMemcpy2DAsync(evec, sizeof(double) * k, d_X, sizeof(double) * ldx, sizeof(double) * k, n,
                              cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess)
            st = ARR_ECUDA;
    }
    cleanup();
    return st;
}

}  // extern "C"
