// Internal declarations of libarrabit (not part of the C-ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/arrabit.h"

// Bounds-checked build (-DARR_CHECK_BOUNDS; build.py variant libarrabit_checked.so): device
// checks of the shared-memory, TMA-destination and staged-CSR indices that trap on a
// violation.  compute-sanitizer is closed on this pool (profiles/r02/); this is its stand-in.
#ifdef ARR_CHECK_BOUNDS
#include <cstdio>
#define ARR_CHECK(cond)                                                                           \
    do {                                                                                          \
        if (!(cond)) {                                                                            \
            printf("ARR_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                            \
            __trap();                                                                             \
        }                                                                                         \
    } while (0)
#else
#define ARR_CHECK(cond) \
    do {                \
    } while (0)
#endif

#define ARR_MAX_W 2048  // largest block width a fused SpMM launch handles
#define ARR_MAX_P 16    // deepest ARR augmentation (the paper uses p <= 3)
constexpr int kPhases = 6;
constexpr int kPhasesAll = 8;  // + 6 = DMMA Gram kernels, 7 = DMMA GEMM kernels (eig_kernel_times)
constexpr int kOmegaCols = 8;  // columns of the re-orthogonality sketch (api.cu arr_core)  // eig_phase_times: filter, arr, residuals, arr.orth, arr.H, arr.eig

// Row-partition plan of one rank (comm.cu; arr_dist in include/arrabit.h).
struct DistPlan {
    int64_t n_global = 0, row_begin = 0, n_ghost = 0;
    std::vector<int> peer;                 // exchange partners (ranks)
    std::vector<int64_t> send_off, recv_off;
    std::vector<char> send_contig;         // rows sent to peer q are one contiguous range
    std::vector<int64_t> send_first;       // first row of that range
    int32_t *send_rows_dev = nullptr;
    double *sendbuf = nullptr, *recvbuf = nullptr;  // packed rows (ld = even ncols)
    int64_t *int_row0 = nullptr, *bnd_row0 = nullptr;
    int32_t *int_len = nullptr, *bnd_len = nullptr;
    int64_t n_int_tiles = 0, n_bnd_tiles = 0;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
    bool cur_direct = true;                // state of the exchange in flight
    int cur_ncols = 0;
    int64_t cur_ld = 0;
};

// Column-partitioned mode (eig_init_colsplit, Survey §8f-3): the outer context holds a
// column context (the full A, this rank's w_loc columns: the filter, no communication)
// and a row context (eig_init_dist on the rank's row block: the ARR projection and the
// residuals), joined by all-to-all transposes of the n x w block (comm.cu).
struct ColSplit {
    std::vector<int64_t> rb, cb;  // [size+1] global row / column boundaries of every rank
    double *sendbuf = nullptr, *recvbuf = nullptr;
    size_t buf_elems = 0;
    arr_ctx *col = nullptr, *row = nullptr;
    double *Xrow = nullptr;       // row-layout block (row context rows x even(w))
    int64_t ldrow = 0;
};

// Stencil-aware filter path (stencil_kernels.cu; eig_set_stencil): A stored as K
// diagonals of a 3x3x3 neighbourhood on an nx x ny x nz grid (x fastest).
struct StencilSlots {
    int K;
    int slot[27];  // bit (dz+1)*9 + (dy+1)*3 + (dx+1) -> DIA column, -1 if absent
};
struct StencilState {
    bool on = false;
    int64_t nx = 0, ny = 0, nz = 0;
    int K = 0, Kpad = 0;
    double *dia = nullptr;  // vmode 0: [n][Kpad] (K rounded up to even: 16-byte rows); vmode 1: the diagonal [n]; owned
    // value mode: 0 = K diagonals (DIA); 1 = constant off-diagonal coefficients coef[slot] and
    // the diagonal per row; 2 = every coefficient constant (no matrix bytes at all)
    int vmode = 0;
    double coef[27] = {};
    int shape = 0, hx = 0, hy = 0;  // stencil_kernels.cu Shape<>: 0 27-pt, 1 7-pt, 2 2-D 5-pt, 3 1-D 3-pt
    int smem_optin = 0;
    // z-slab of a row partition (eig_init_dist): nz = the owned planes; gz_lo / gz_hi = 1 when
    // the plane below / above is a ghost plane (the block's rows n .. n + (gz_lo + gz_hi) nx ny,
    // lower plane first: the ghost rows sorted by global id)
    int gz_lo = 0, gz_hi = 0;
    // the plan's boundary tiles (rows with a ghost column) are exactly the slab's first / last
    // plane: those rows may run on the CSR kernels after the exchange (api.cu spmm_x)
    bool bnd_is_ends = false;
};
// One launch of the stencil kernel (kernel parameter, __grid_constant__).
struct StencilLaunch {
    CUtensorMap tm_in, tm_prev, tm_xa, tm_val;  // TMA descriptors (64-byte aligned)
    const double *Yin, *Yprev, *Xa;
    double *Yout;
    int64_t ld_in, ld_prev, ld_out, ld_xa;
    double alpha, shift, beta, gxa;
    const double *colscale;  // lazy MPM column scale (SpmmArgs::colscale) or nullptr
    int scale_mode;          // 1: scale the output, 2: scale the Y_{j-1} term
    double *partials;
    const double *val;
    double coef[27];  // constant coefficients by DIA slot (vmode 1: off-diagonal slots; vmode 2: all)
    int vmode, Pxe;   // value mode (StencilState); the diagonal's box width (Px rounded up to even)
    int64_t nitems;
    int w, wv, K, Kpad;
    int nx, ny, nz;
    int gz_lo, gz_hi;  // ghost planes below / above the nz owned planes (StencilState)
    int z0, z1;        // output planes of this launch (z-chunks of [z0, z1))
    int zstep;         // distance of consecutive z-chunks' first planes (Lz; z1 - 1 - z0 for the two end planes)
    int Px, Py, Lz, npx, npy, nzc, npan, pwv, NS;
    int box_x, box_y, hx, hy;
    int pm;  // 1: panel-major work-item order (stencil_kernels.cu decode_item)
    int dyn;  // 1: work items from the atomic ticket `sched` (launches without column sums)
    unsigned long long *sched;  // [2] ticket + finished-CTA count (self-resetting; the context's)
    int ypol, spol, opol;  // L2 eviction policies of the Y_j boxes / once-read operands / stores
};

struct arr_ctx {
    // problem
    arr_csr A;
    int32_t k, w, p, d;
    cudaStream_t stream;
    int num_sms;
    int max_row_nnz;  // longest CSR row (selects the SpMM chunk size)
    int tile_rows;    // SpMM rows per tile in natural order (1..64; env ARRABIT_TILE)
    int col_split;    // column vectors per SpMM thread (1 default; env ARRABIT_SPLIT, tuning)
    // deflation (solve_deflate): locked vectors the augmentation blocks are projected against
    const double *defl_Q;
    int64_t defl_ld;
    int defl_n;
    // eig_set_mode: +1 = k largest eigenpairs of A, -1 = k smallest (the solver runs on -A)
    int sign;
    // polynomial filter (eig_set_filter): 0 = T_d, 1 = psi_d (Chebyshev coefficients coef[0..d])
    int filter_kind;
    std::vector<double> coef;
    // interval
    double a, b;
    bool have_interval;
    // workspace (owned)
    double *T;        // n x w scratch (filter ping-pong, ARR W)
    double *Q;        // n x m ARR basis, ld = m
    double *part;     // Gram split partials / column-norm partials
    size_t part_elems;
    double *small;    // dense m x m buffers (H, V, B ...)
    double *evals;    // [m]
    double *vecw;     // [2*ARR_MAX_W] column norms / shifts / scales
    // lazy MPM normalisation (filter_core normalize = 2): lazy[0, mw) = the pending column
    // norms of lazy_X, lazy[mw, 2 mw) = their reciprocals D (mw = ARR_MAX_W + 2)
    double *lazy;
    const double *lazy_X;
    bool lazy_pending;
    int *dinfo;       // cuSOLVER info + rank counters
    unsigned long long *sched;  // [2] SpMM tile ticket (zeroed at init, self-resetting)
    double *omega;              // [w x kOmegaCols] seeded Gaussian sketch of the ARR re-orthogonality check
    double *racc;               // [2 x w x w] CholeskyQR factor R of the last augmentation block (R23)
    const int64_t *tile_row0;   // eig_set_schedule (borrowed device arrays) or nullptr
    const int32_t *tile_len;
    int64_t ntiles;
    double *solver_work;
    int solver_lwork;
    void *trtri_dwork;      // cusolverDnXtrtri device workspace
    size_t trtri_dbytes;
    std::vector<char> trtri_hwork;
    int orth_mode;          // 0 = shifted CholeskyQR3 (fallback SVQB), 1 = SVQB only
    cusolverDnHandle_t solver;
    size_t ws_bytes;
    // filter degree loop as a CUDA graph (api.cu run_degrees)
    cudaGraphExec_t g_exec;
    alignas(8) unsigned char g_key[128];
    bool g_key_set;
    uint64_t g_kernels;
    int64_t g_spmm;
    int g_nblk;
    const char *g_last_kernel;
    // bookkeeping
    const char *last_kernel;  // name of the kernel the last fused SpMM launched (eig_last_spmm_kernel)
    uint64_t launches;
    int64_t spmm_blocks;
    arr_status poisoned;
    std::string err;
    // phase timing (eig_set_timing)
    bool timing;
    std::vector<cudaEvent_t> ev_pool;
    int ev_next;
    struct Pending { int phase, e0, e1; int64_t count; double work; };
    std::vector<Pending> pending;
    double phase_ms[kPhasesAll];
    int64_t phase_cnt[kPhasesAll];
    double phase_work[kPhasesAll];  // algorithmic flops of the timed DMMA launches (phases 6, 7)
    // multi-GPU (eig_init_dist): communicator, partition plan, allreduce staging
    arr_comm *comm;
    int nranks;  // size of comm (1 without one)
    DistPlan plan;
    StencilState st;
    ColSplit *cs;  // column-partitioned outer context (nullptr otherwise)
    // row context of a column split: its ARR SpMMs run in the column layout (transpose,
    // local SpMM with the replicated A on the column context, transpose back)
    ColSplit *cs_link;
    arr_ctx *cs_outer;
    double *stage;
    size_t stage_elems;
    // pinned host staging
    double *h_stage;   // [m + 2*ARR_MAX_W + 16]
    int *h_istage;     // [16]
};

// ---------------------------------------------------------------- SpMM family
struct SpmmArgs {
    const int64_t *row_ptr;
    const int32_t *col;
    const double *val;
    int64_t n;
    int64_t nnz;           // entries of A (bounds the CSR prefetch)
    int32_t w;
    const double *Yin;     // gathered operand Y_j
    int64_t ld_in;
    const double *Yprev;   // Y_{j-1} (may alias Yout) or nullptr
    int64_t ld_prev;
    double *Yout;          // output or nullptr (no store)
    int64_t ld_out;
    double alpha, shift, beta;
    const double *colshift;  // per-column shift (overrides shift) or nullptr
    const double *Xa;        // optional fourth operand: Yout += gxa * Xa (interpolant filter), or nullptr
    int64_t ld_xa;
    double gxa;
    // lazy MPM normalisation (Survey §8a A2, p_d(A)(X D) = p_d(A) X D): per-column scale D,
    // scale_mode 1 = the output is D * (...) (the first degree), 2 = the Y_{j-1} term is
    // beta D y_prev (the second degree); 0 / nullptr = none
    const double *colscale;
    int scale_mode;
    double *partials;        // [gridDim.x * w] column sums of squares of the output, or nullptr
    unsigned long long *sched;  // [2] dynamic tile ticket + finished-CTA count (self-resetting)
    const int64_t *tile_row0;   // optional processing order: tile t = rows [tile_row0[t], +tile_len[t])
    const int32_t *tile_len;
    int64_t ntiles;
};

// Per-kernel-instantiation cache of the dynamic shared-memory attribute and the
// occupancy at that size; the mutex makes it safe for the host threads of an
// in-process rank group (comm_init_local_group) that launch concurrently.
struct LaunchCache {
    std::mutex mu;
    int occ = -1;
    size_t smem = 0;
};
template <class Kern>
int cached_occupancy(LaunchCache &lc, Kern kern, int threads, size_t smem) {
    std::lock_guard<std::mutex> lk(lc.mu);
    if (lc.occ < 0 || lc.smem != smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int o = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem);
        lc.occ = o > 0 ? o : 1;
        lc.smem = smem;
    }
    return lc.occ;
}

// Launch the fused SpMM: Yout = alpha*(A Yin - shift*Yin) + beta*Yprev.
// Returns the grid size used (number of partial rows written if partials != nullptr).
int launch_spmm(arr_ctx *c, const SpmmArgs &a);
// stencil path (stencil_kernels.cu): -1 when it does not apply to this launch
// z0 / z1: the output planes of this launch (z1 < 0: all owned planes); ends_only: just the
// planes z0 and z1 - 1 (a z-slab's two planes next to the ghost planes, one launch)
int launch_spmm_stencil(arr_ctx *c, const SpmmArgs &a, int z0 = 0, int z1 = -1, bool ends_only = false);
arr_status stencil_setup(arr_ctx *c, int64_t nx, int64_t ny, int64_t nz, int gz_lo = 0, int gz_hi = 0);
void stencil_release(arr_ctx *c);
// out[col] = sqrt(sum_b partials[b*w + col]) ; if rel != nullptr: out /= max(1,|rel|)
void launch_colnorm_finalize(arr_ctx *c, const double *partials, int nblk, int32_t w, double *out,
                             const double *mu_div);
// out[col] = sum_b partials[b*w + col] (no root; multi-GPU: allreduced, then launch_colnorm_root)
void launch_colsum(arr_ctx *c, const double *partials, int nblk, int32_t w, double *out);
// x[col] = sqrt(x[col]) / (mu_div ? max(1,|mu_div[col]|) : 1)
void launch_colnorm_root(arr_ctx *c, double *x, int32_t w, const double *mu_div);
// X[i, col] *= 1/norm[col] (in place) or Out = In / norm
void launch_scale_cols(arr_ctx *c, const double *In, int64_t ld_in, double *Out, int64_t ld_out,
                       int64_t n, int32_t w, const double *norms);
void launch_recip(arr_ctx *c, const double *x, int32_t w, double *out);  // out = 1 / x
void launch_gershgorin(arr_ctx *c, double *partial, int *nblk_out);
void launch_rowlen_max(arr_ctx *c, int *dev_out);
// exact-cover check of a schedule: bad = 1 unless every row is covered once
void launch_schedule_check(arr_ctx *c, const int64_t *row0, const int32_t *len, int64_t ntiles, int *marks,
                           int *bad);
void launch_min_finalize(arr_ctx *c, const double *partial, int nblk, double *out);

// ---------------------------------------------------------------- multi-GPU (comm.cu)
// All are no-ops when the context has no communicator or a group of one.
// op: 0 sum, 1 min, 2 max.  Results are identical on every rank.
arr_status comm_allreduce(arr_ctx *c, double *buf, size_t count, int op);
arr_status comm_bcast(arr_ctx *c, double *buf, size_t count, int root);
arr_status comm_halo_begin(arr_ctx *c, const double *Y, int64_t ld, int ncols);
arr_status comm_halo_end(arr_ctx *c, double *Y);
arr_status comm_setup_plan(arr_ctx *c, const arr_dist *d, arr_comm *m);
// dir 0: column layout (n x w_loc, ld lds) -> row layout (rows of this rank x w, ld ldd);
// dir 1: back.  Collective over the column split's communicator.
arr_status comm_transpose(arr_ctx *c, const ColSplit &S, int dir, const double *src, int64_t lds, double *dst,
                          int64_t ldd);
void comm_free_plan(arr_ctx *c);

// ---------------------------------------------------------------- dense (DMMA)
int gram_nsplit(int64_t n, int32_t m1, int32_t m2, int num_sms, bool sym);
// phase timing (eig_set_timing): an event on the context stream (-1 when timing is off) and a
// pending (phase, start, end, count, algorithmic flops) interval resolved at the next sync
inline int t_mark(arr_ctx *c) {
    if (!c->timing) return -1;
    if (c->ev_next == (int)c->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return -1;
        c->ev_pool.push_back(e);
    }
    const int i = c->ev_next++;
    cudaEventRecord(c->ev_pool[i], c->stream);
    return i;
}
inline void t_add(arr_ctx *c, int phase, int e0, int e1, int64_t count, double work = 0.0) {
    if (e0 >= 0 && e1 >= 0) c->pending.push_back({phase, e0, e1, count, work});
}
// sym_result: X != Y but X^T Y is symmetric in exact arithmetic (U^T (A U)): only the tiles on
// or above the diagonal are computed and the result is their exact mirror
void launch_gram(arr_ctx *c, const double *X, int64_t ldx, int32_t m1, const double *Y, int64_t ldy,
                 int32_t m2, int64_t n, double *G, int64_t ldg, double *partials, bool sym_result = false);
// upper != 0: B is upper triangular (exact zeros below the diagonal are skipped)
void launch_gemm(arr_ctx *c, double alpha, const double *X, int64_t ldx, int32_t m1, const double *B,
                 int64_t ldb, int32_t m2, double beta, const double *Cin, int64_t ldc, double *Out,
                 int64_t ldo, int64_t n, int upper = 0);
// small dense helpers (single CTA-ish kernels)
void launch_svqb_prep(arr_ctx *c, const double *G, int32_t w, double *D, double *Gs);
void launch_svqb_build(arr_ctx *c, const double *D, const double *Vcm, const double *lam, int32_t w,
                       double tau, double *B, int *rank_out);
void launch_symmetrize(arr_ctx *c, double *H, int32_t m, int32_t bw);
void launch_ritz_select(arr_ctx *c, const double *Vcm, int32_t m, int32_t wsel, double *Vsel);
void launch_copy_rows(arr_ctx *c, const double *src, int64_t lds, double *dst, int64_t ldd, int64_t n,
                      int32_t w);
void launch_check_norms(arr_ctx *c, const double *norms, int32_t w, int *bad);
void launch_chol_prep(arr_ctx *c, const double *G, int32_t w, double shift, double *D, double *Gs);
void launch_chol_build(arr_ctx *c, const double *D, const double *Rinv_cm, int32_t w, double *B, const double *Rdiag,
                       double rank_thr, int *rank_out);
void launch_diag_copy(arr_ctx *c, const double *A_cm, int32_t w, double *d);
// Rnew = (Rs diag(D)^-1) Rold (first: Rs diag(D)^-1): the inverse of one CholeskyQR pass's
// transform B = diag(D) Rs^-1 folded into the accumulated factor (Rs column-major upper,
// Rold / Rnew row-major upper, w x w)
void launch_chol_racc(arr_ctx *c, const double *Rs_cm, const double *D, int32_t w, const double *Rold, double *Rnew,
                      bool first);
// H[r0 + a][c0 + b] = R[b][a] (R row-major w x w upper, H row-major, ld m)
void launch_put_rt(arr_ctx *c, const double *R, int32_t w, double *H, int64_t ldh);

void launch_dev_from_identity(arr_ctx *c, const double *M_cm, int32_t w, double *out);
void launch_maxabs(arr_ctx *c, const double *x, int64_t count, double *out);
void launch_mirror_upper(arr_ctx *c, double *M, int32_t w);  // row-major upper -> lower
void launch_add_diag(arr_ctx *c, double *M, int32_t w, int64_t ld, double v);
