/*
 * arrabit.h — C-ABI of the B200 (sm_100a) hot path of ARRABIT-MPM,
 * Wen & Zhang, "Block algorithms with augmented Rayleigh-Ritz projections for
 * large-scale eigenpair computation", arXiv 1507.06078.
 * Citations "P:n" are lines of the paper text; section / equation /
 * algorithm names follow the paper's LaTeX labels.
 *
 * Conventions (every entry point):
 *  - Every call returns arr_status; ARR_OK == 0.  No exception crosses the ABI;
 *    a message for the last failure is kept per context (eig_last_error).
 *  - Ownership: the CSR arrays and every block passed in are CALLER-OWNED DEVICE
 *    memory and must outlive the context.  eig_init allocates the context's own
 *    workspace (one n x w scratch block, the n x (p+1)w ARR basis, Gram partials
 *    and small dense buffers); eig_destroy frees it.  No other call allocates.
 *  - Layout: blocks are ROW-MAJOR n x ncols fp64 with leading dimension ld >= ncols
 *    (elements).  Row i of a block starts at base + i*ld.  When ncols and ld are
 *    even and the base is 16-byte aligned the kernels use 128-bit accesses;
 *    otherwise a scalar path runs (same results).
 *  - CSR: full symmetric pattern stored (both triangles), row_ptr int64 [n+1],
 *    col_idx int32 [nnz] (sorted or not), val fp64 [nnz].
 *  - Streams: everything is enqueued on the stream given to eig_init (a
 *    cudaStream_t passed as void*; NULL = legacy default stream).  Calls that
 *    return host data (ritz_host, rank, res_host, a_out, the solve outputs)
 *    synchronise that stream; all others are asynchronous.
 *  - Errors: bad sizes / pointers / interval -> ARR_EINVAL (context stays usable).
 *    A CUDA, cuSOLVER or NCCL failure poisons the context: every later call returns
 *    the same code.  A zero or non-finite column norm after filtering ->
 *    ARR_ENUMERIC.  Rank loss is NOT an error; *rank reports it.
 *  - Determinism: fixed reduction trees, no floating-point atomics.  Identical
 *    inputs on the same GPU model give bitwise identical outputs.
 */
#ifndef ARRABIT_H
#define ARRABIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct arr_ctx arr_ctx;

typedef enum {
    ARR_OK = 0,
    ARR_EINVAL = 1,
    ARR_ENOMEM = 2,
    ARR_ECUDA = 3,
    ARR_ECUSOLVER = 5,
    ARR_ENCCL = 6,
    ARR_ENUMERIC = 7
} arr_status;

/* Sparse symmetric A (borrowed device arrays). */
typedef struct {
    int64_t n;               /* rows = columns of A                          */
    int64_t nnz;             /* stored entries                                */
    const int64_t *row_ptr;  /* device [n+1]                                  */
    const int32_t *col_idx;  /* device [nnz], 0 <= col < n                    */
    const double *val;       /* device [nnz]                                  */
} arr_csr;

/* ---------------------------------------------------------------- multi-GPU (A7)
 * Row partition (north star "A is row-partitioned with X rows
 * co-located.  An NCCL halo exchange (or all-gather of X for irregular
 * sparsity) runs before each SpMM ..., and a k x k NCCL allreduce handles the
 * Gram blocks").  Rank r owns the contiguous global rows
 * [row_begin, row_begin + A.n) of A and of every n x w block.  Its local CSR
 * (arr_csr with n = owned rows) numbers columns locally: 0 .. A.n-1 are the
 * owned rows, A.n .. A.n + n_ghost - 1 the ghost rows (rows owned elsewhere that
 * its rows reference), grouped by owner in peer order.  EVERY block passed to
 * a distributed context has A.n + n_ghost rows; the ghost rows are scratch the
 * library fills before each SpMM.  A must be structurally symmetric, so the rows
 * rank r sends to peer q are exactly q's ghost rows from r (in the same order).
 * paper_1507_06078_b200/partition.py builds this plan from a global CSR. */
typedef struct arr_comm arr_comm;

typedef struct {
    int64_t n_global;          /* rows of the global A                                   */
    int64_t row_begin;         /* first owned global row                                 */
    int64_t n_ghost;           /* ghost rows appended after the owned rows               */
    int32_t npeers;            /* exchange partners                                      */
    const int32_t *peer;       /* host [npeers] ranks (!= own rank)                      */
    const int64_t *send_off;   /* host [npeers+1] offsets into send_rows                 */
    const int32_t *send_rows;  /* host [send_off[npeers]] local owned rows sent to peer q */
    const int64_t *recv_off;   /* host [npeers+1]; ghost rows from peer q are local rows
                                  A.n + recv_off[q] .. A.n + recv_off[q+1]-1;
                                  recv_off[npeers] == n_ghost                            */
    const int64_t *int_row0;   /* host [n_int_tiles] interior row tiles (rows with no ghost
                                  column; computed while the exchange is in flight)      */
    const int32_t *int_len;    /* 1..64 rows each                                        */
    int64_t n_int_tiles;
    const int64_t *bnd_row0;   /* host [n_bnd_tiles] boundary row tiles (computed after   */
    const int32_t *bnd_len;    /* the exchange); interior + boundary = every owned row once */
    int64_t n_bnd_tiles;
} arr_dist;

/* NCCL communicator of one rank (one process per GPU; call with the rank's
 * device current).  id: 128 bytes from comm_get_nccl_id on one rank, broadcast
 * to all (e.g. with torch.distributed).  Collective over the size ranks. */
arr_status comm_get_nccl_id(unsigned char *id_out /* [128] */);
arr_status comm_init_nccl(arr_comm **out, const unsigned char *id, int32_t rank, int32_t size);
/* size communicators for size ranks driven by size host threads of ONE
 * process (any devices it can address; the same GPU is allowed).  The same
 * exchange, reductions and broadcasts as NCCL, done with device copies and
 * fixed-order reduction kernels ordered by host barriers and stream events.
 * out: host array [size].  Used to test the distributed path on one GPU. */
arr_status comm_init_local_group(arr_comm **out, int32_t size);
arr_status comm_rank_size(const arr_comm *m, int32_t *rank, int32_t *size);
/* Destroy after every context using it is destroyed. */
arr_status comm_destroy(arr_comm *m);

/* Options / report of the fixed-parameter driver eig_solve. */
typedef struct {
    double tol;      /* outer stop: max_i res_i <= tol (Eq. out-stop)   */
    int32_t maxit;   /* maximum outer iterations                        */
    int32_t s_max;   /* cap of the sweeps-per-ARR rule (R6)                 */
    int32_t exits;   /* the paper's extra stop rules, a bit mask, 0 = off
                        (R10): 1 = (ii) max res not reduced over three
                        consecutive outer iterations; 2 = (iii) max res < (1 + 9h/k) tol,
                        h = #{res_i < 0.1 tol}                                       */
    int32_t inner;   /* sweeps between ARR steps: 0 = the dynamic-range rule (R6),
                        1 = the paper's rcond rule (check rcond(X^T X) every 5
                        sweeps, at most 10 times; stop at rc <= tol or rc/rc_prev > 0.99) */
    int32_t adapt;   /* the paper's adaptive parameters, a bit mask, 0 = fixed p and d:
                        1 = p starts at 1 and grows by Eq. block up to the
                        context's p; 2 = d starts at 3 and is re-chosen after every ARR by
                        Eqs. hat-d / degree, the context's d as d_max;
                        4 = continuation + deflation (locking) of converged pairs, the
                        paper's b update at continuation (R19);
                        bit 4 runs fixed p / d MPM sweeps with the dynamic-range rule and
                        returns ARR_EINVAL combined with bits 1/2, gn, inner or exits   */
    int32_t gn;      /* inner solver: 0 = MPM (filter + column normalisation),
                        1 = Gauss-Newton (Alg. Arrabit2: Y = X (X^T X)^{-1},
                        Z = rho_d(A) Y, X = Z - X (Y^T Z - I)/2); needs p >= 1; a step
                        whose X^T X is not positive definite returns ARR_ENUMERIC   */
    int64_t grid[3]; /* eig_solve_host only: {nx, ny, nz} != 0 declares A a stencil operator
                        (eig_set_stencil on the internal context); {0,0,0}: CSR kernels  */
    double *log;     /* optional host [log_cap x ARR_LOG_FIELDS]: one row per outer iteration
                        {outer, sweeps s, a, b, mu_1 that set s, max res, p, d, locked, tol_t,
                        mu_k, mu_w} - the driver's decisions and the Ritz values they are
                        taken from, for checking them against the rules                  */
    int32_t log_cap; /* rows available in log (0: no log)                                */
    double range_digits; /* D of the dynamic-range rule (inner = 0): s = clamp(floor(D /
                        log10 |T_d((mu_1 - c)/e)|), 1, s_max); 0 = the default D = 12
                        (R6)                                                   */
} arr_solve_opts;
#define ARR_LOG_FIELDS 12

typedef struct {
    int32_t converged;   /* 1 if max res <= tol                                   */
    int32_t outer;       /* outer iterations done                                 */
    int32_t sweeps;      /* MPM sweeps done (each = d filter degrees)            */
    int32_t last_rank;   /* numerical rank reported by the last ARR               */
    double maxres;       /* final max_i res_i                                     */
    double a, b;         /* final filter interval                                 */
    int64_t spmm_blocks; /* block SpMMs issued (filter degrees + ARR + residuals) */
    int32_t exit_rule;   /* why the outer loop ended: 1 max res <= tol, 2 rule (ii),
                            3 rule (iii), 0 maxit                                   */
    int32_t p_final;     /* augmentation depth of the last ARR                      */
    int32_t d_final;     /* filter degree of the last sweeps                        */
    int32_t locked;      /* pairs locked by deflation (adapt bit 4)                 */
} arr_solve_info;

/* ---------------------------------------------------------------- lifecycle
 * eig_init: create a context for A with k wanted pairs, block width w = k,
 * ARR augmentation depth p (Eq. S:ARR) and Chebyshev degree d
 * (Eq. cheby-poly).  Requires 1 <= k, 0 <= p <= 16, 1 <= d, (p+1)k < n
 * (Alg. ARR input), n < 2^31.  stream: cudaStream_t or NULL.
 * Allocates the workspace described above (ARR_ENOMEM if it does not fit). */
arr_status eig_init(arr_ctx **out, const arr_csr *A, int32_t k, int32_t p, int32_t d, void *stream);
/* Same with an explicit block width w >= k: w - k guard vectors (P:1291-1299,
 * "the number of columns in iterate matrix X to k+q"); (p+1)w < n.  Blocks
 * passed to filter_step / arr_project / eig_solve are then n x w; residuals and
 * the stop rule use the k leading pairs; b = mu_{w+1} (R3). */
arr_status eig_init_w(arr_ctx **out, const arr_csr *A, int32_t k, int32_t w, int32_t p, int32_t d, void *stream);
/* Distributed context (collective over the ranks of comm): A_local is this
 * rank's local CSR (see arr_dist), k/w/p/d as eig_init_w with (p+1)w < n_global.
 * Every later call on the context is collective: all ranks make the same
 * sequence of calls.  Gram products, column norms, residual norms, Ritz values
 * and eigenvalues are reduced over ranks and identical on every rank; blocks
 * hold the owned rows (+ ghost scratch rows).  comm == NULL or a group of one
 * behaves as eig_init_w.  The plan's host arrays are copied. */
arr_status eig_init_dist(arr_ctx **out, const arr_csr *A_local, int32_t k, int32_t w, int32_t p, int32_t d,
                         const arr_dist *dist, arr_comm *comm, void *stream);
/* Column-partitioned context (Survey §8f-3), collective over the ranks of comm.
 * MPM filters every column independently ("x_i <- rho(A) x_i"), so with A
 * replicated a rank filters its column slice with NO communication; only the ARR
 * projection (Alg. ARR) needs the whole block.  Rank r owns columns
 * [col_begins[r], col_begins[r+1]) of every n x w block it passes (X: n x w_r, all n
 * rows) and, for the ARR projection and the residuals, an internal row-partitioned
 * context (as eig_init_dist) on rows [row_begins[r], row_begins[r+1]): A_rows / rows
 * are that row block's local CSR and exchange plan (partition.colsplit_plan builds
 * them).  Between the two, the block moves by one all-to-all transpose each way
 * (comm.cu comm_transpose; 2 n w doubles per outer iteration in total over all
 * ranks, against d x sweeps halo / all-gather exchanges of the row partition).
 * A_full: the whole matrix on every rank.  row_begins / col_begins: host [size+1],
 * identical on every rank, col_begins[size] = w.  Supported calls: filter_step
 * (local), arr_project(_p) and residuals (column slices in and out), eig_solve
 * (fixed parameters: adapt / gn / inner / exits -> ARR_EINVAL), the interval /
 * degree / filter / mode / stencil / schedule setters (applied to the column
 * context), spmm (whole A on this rank's columns), timing; gram / gemm /
 * orthonormalize return ARR_EINVAL. */
arr_status eig_init_colsplit(arr_ctx **out, const arr_csr *A_full, int32_t k, int32_t w, int32_t p, int32_t d,
                             const arr_csr *A_rows, const arr_dist *rows, const int64_t *row_begins,
                             const int64_t *col_begins, arr_comm *comm, void *stream);
arr_status eig_destroy(arr_ctx *c);
const char *eig_last_error(const arr_ctx *c);
size_t eig_workspace_bytes(const arr_ctx *c);
/* Number of kernels this context has launched so far (a replayed CUDA graph
 * counts every kernel node).  Library calls (cuSOLVER) are not counted. */
uint64_t eig_launch_count(const arr_ctx *c);
/* Phase timing (CUDA events on the context stream, resolved at the stream
 * syncs the calls already make).  on != 0 enables it and zeroes the totals.
 * eig_phase_times synchronises the stream and returns, for phase
 * 0 = filter degree kernels (the d fused SpMM launches of each filter_step),
 * 1 = arr_project, 2 = residuals, and the parts of arr_project 3 = building
 * the orthonormal block-Krylov basis, 4 = H = Q^T A Q, 5 = small dense eig:
 * ms[6] total device milliseconds and counts[6] (phase 0: degree launches;
 * others: calls). */
arr_status eig_set_timing(arr_ctx *c, int32_t on);
arr_status eig_phase_times(arr_ctx *c, double *ms, int64_t *counts);
/* The FP64 DMMA kernels alone (with eig_set_timing on; events around each launch,
 * the split reduction excluded): index 0 = the Gram kernels (X^T Y, Alg. RR / ARR
 * products P:219-224), 1 = the GEMM kernels (X B): total device ms,
 * ALGORITHMIC flops (2 n m1 m2; a symmetric Gram n m (m+1); an upper-triangular B
 * 2 n sum_c min(c+1, m1)) and launch counts since timing was enabled.  Synchronises
 * the stream.  Column-split contexts report their ARR (row) context. */
arr_status eig_kernel_times(arr_ctx *c, double *ms /* [2] */, double *flops /* [2] */,
                            int64_t *launches /* [2] */);

/* ---------------------------------------------------------------- A0: interval
 * a_out = min_i (A_ii - sum_{j!=i} |A_ij|), the Gershgorin lower bound used in
 * place of the paper's eigs estimate of lambda_n (R3). */
arr_status eig_gershgorin_lower(arr_ctx *c, double *a_out);
/* Set the damped interval [a,b] (Eq. rhod):
 * c = (a+b)/2, e = (b-a)/2.  a >= b -> ARR_EINVAL. */
arr_status eig_set_interval(arr_ctx *c, double a, double b);
/* Optional processing order of the rows of A for every SpMM of this context
 * (results are unchanged: only the order in which rows are computed moves,
 * to shorten the L2 reuse distance of gathered rows).  Tile t is
 * the contiguous row range [tile_row0[t], tile_row0[t] + tile_len[t]),
 * 1 <= tile_len[t] <= 64; tiles are processed in increasing t.  The tiles must
 * cover every row exactly once (checked here with a device pass over the
 * scratch block; ARR_EINVAL otherwise; synchronises the stream).  Device
 * arrays, borrowed (must outlive the context or the next call).
 * tile_row0 == NULL restores natural order. */
arr_status eig_set_schedule(arr_ctx *c, const int64_t *tile_row0, const int32_t *tile_len, int64_t ntiles);
/* Declare A a stencil operator on an nx x ny x nz grid (row i = x + nx (y + ny z),
 * x fastest): every row's columns sorted ascending and within the 3x3x3
 * neighbourhood of its grid point (the finite-difference operators of the paper's
 * test set; cfg 1-3, 5).  The pattern is verified on the device
 * (ARR_EINVAL if it does not hold or nx*ny*nz != n); then A is stored once more as K
 * diagonals (DIA, K = number of neighbour offsets present, 8 K n bytes allocated
 * here: the one allocation after eig_init; ARR_ENOMEM if it does not fit) and every
 * fused SpMM of the context without a per-column shift runs the stencil-aware
 * 2.5-D blocked kernel: same per-row FMA order, so outputs are
 * bitwise those of the CSR kernels.  nx = ny = nz = 0 switches back to CSR and
 * frees the copy.  Synchronises the stream.
 * Row-partitioned contexts (eig_init_dist): (nx, ny, nz) is this rank's z-slab of whole
 * grid planes (nx ny nz = the owned rows) and its ghost rows must be exactly the
 * neighbouring plane below (received from lower ranks, first) and / or above (the
 * layout partition.py builds for bounds_planes); anything else is ARR_EINVAL.  Each
 * fused SpMM then runs the stencil kernel on the planes that touch no ghost plane
 * while the halo exchange is in flight and on the slab's first / last plane after it
 * (the same sums: bitwise the one-GPU result).  Column-split contexts declare the
 * whole grid (the column context holds all of A). */
arr_status eig_set_stencil(arr_ctx *c, int64_t nx, int64_t ny, int64_t nz);
/* K of the active stencil path (0 = the CSR kernels). */
int32_t eig_stencil_active(const arr_ctx *c);
/* Bytes of A the stencil path reads per row and column panel: eig_set_stencil detects
 * constant coefficients (every neighbour slot's value the same on all rows whose neighbour
 * is in the grid, as in the finite-difference operators of P:1624-1627) and then keeps
 * only the diagonal (8 bytes per row; needs nx even) or nothing (0: all coefficients
 * constant, the operator applied matrix-free); otherwise the K diagonals (8 K).  -1 when
 * no stencil is active.  ARRABIT_ST_VMODE=0 forces the K diagonals. */
int32_t eig_stencil_abytes(const arr_ctx *c);
/* Name of the kernel the context's last fused SpMM launched (static string; "" if none). */
const char *eig_last_spmm_kernel(const arr_ctx *c);
/* Change the degree d used by filter_step (1 <= d). */
arr_status eig_set_degree(arr_ctx *c, int32_t d);
/* Which end of the spectrum: smallest = 0 (default): the k algebraically largest
 * eigenpairs; smallest != 0: the k algebraically smallest (the paper's
 * second mode, Table 6) by running the whole method on -A.  In that mode the
 * interval calls (eig_gershgorin_lower, eig_set_interval, the filter) refer to the
 * spectrum of -A, while eigenvalues and Ritz values returned by eig_solve /
 * arr_project and mu passed to residuals are those of A (ascending: smallest first).
 * Clears the interval. */
arr_status eig_set_mode(arr_ctx *c, int32_t smallest);
/* Polynomial of filter_step / eig_solve: kind 0 = the classic Chebyshev polynomial
 * T_d of the mapped matrix (default, Eq. cheby-poly); kind 1 = the
 * paper's default filter rho_d(t) = psi_d((2t - a - b)/(b - a)), psi_d the degree-d
 * Chebyshev interpolant of max(0, t)^{10 d} at the Chebyshev points of the second
 * kind (Section 5), applied in the Chebyshev basis by Clenshaw's
 * recurrence (R18; one fused SpMM per degree with X as a fourth operand:
 * 12 nnz + 8(n+1) + 32 n w bytes per degree).  Uses the basis buffer as a second
 * scratch block (ARR_EINVAL in a lean context with p = 0). */
arr_status eig_set_filter(arr_ctx *c, int32_t kind);

/* ---------------------------------------------------------------- A1 + A2
 * X <- T_d((A - cI)/e) X by the three-term recurrence
 *   Y_0 = X, Y_1 = (A Y_0 - c Y_0)/e, Y_{j+1} = (2/e)(A Y_j - c Y_j) - Y_{j-1}
 * (Eq. cheby-poly P:377-383 on the map of Eq. rhod; Alg. Arrabit2
 * line P:1486), one fused SpMM kernel per degree.  If normalize == 1, every
 * column is then scaled to unit 2-norm (MPM) and, when
 * colnorm_dev != NULL, the pre-normalisation norms are written there (device
 * [w]).  normalize == 2 (lazy, Survey §8a A2): the norms are computed and checked
 * but X is left unscaled; the scale D = 1/norm is kept pending and an IMMEDIATELY
 * following filter_step on the same X folds it into its first two degrees
 * (p_d(A)(X D) = p_d(A) X D), saving one pass over the block; any other call on the
 * context drops it (X then simply stays unnormalised).  d odd, the interpolant filter
 * or colnorm_dev != NULL normalise eagerly instead.  X: device n x w, row-major,
 * ldx >= w.  Uses the context scratch block.  Returns ARR_ENUMERIC if a norm is zero
 * or not finite (checked only when normalize != 0; this synchronises the stream);
 * ARR_EINVAL for normalize outside {0, 1, 2}. */
arr_status filter_step(arr_ctx *c, double *X, int64_t ldx, int32_t normalize, double *colnorm_dev);

/* ---------------------------------------------------------------- A3 (test hook)
 * Y = alpha (A - shift I) X for ncols columns (ncols <= 2048).  X, Y device,
 * row-major, must not alias.  Always A itself (also in eig_set_mode smallest).
 * On a distributed context the call is collective: the ghost rows of X are
 * exchanged first (they are overwritten), then the owned rows of Y computed. */
arr_status spmm(arr_ctx *c, double alpha, double shift, const double *X, int64_t ldx,
                double *Y, int64_t ldy, int32_t ncols);

/* ---------------------------------------------------------------- A4
 * Tall-skinny fp64 products on DMMA tensor cores (mma.sync m8n8k4.f64).
 * gram:  G = X^T Y, X n x m1, Y n x m2, G device row-major m1 x m2 (ldg).
 *        Split over rows, fixed-order reduction (deterministic).  m1 * m2 must
 *        fit the context's partial-sum buffer (>= max(16 m w, 4096 max(m, 2048))
 *        doubles, m = (p+1)w), else ARR_EINVAL.
 * gemm:  Out = beta*Cin + alpha * X B, X n x m1, B device row-major m1 x m2 (ldb),
 *        Cin/Out n x m2.  Cin may equal Out; X must not alias Out.       */
arr_status gram(arr_ctx *c, const double *X, int64_t ldx, int32_t m1, const double *Y, int64_t ldy,
                int32_t m2, double *G, int64_t ldg);
arr_status gemm(arr_ctx *c, double alpha, const double *X, int64_t ldx, int32_t m1, const double *B,
                int64_t ldb, int32_t m2, double beta, const double *Cin, int64_t ldc, double *Out,
                int64_t ldo);

/* Orthonormalise the ncols (<= w) columns of X in place: shifted CholeskyQR3
 * (Gram X^T X on DMMA, column equilibration, shift 11(n c + c(c+1)) u c, potrf,
 * trtri, X <- X D R^{-1}; two unshifted passes follow, the third skipped when the
 * second factor is within 1e-6 of I), falling back to two SVQB passes
 * (X <- X D V L^{-1/2}) if a Cholesky factorisation fails.  The span is that of X
 * plus, if X is rank deficient, directions from its rounding noise (Alg. RR
 * step 1, "orthonormalize Z").  *rank = number of R_ii^2 above
 * 100 x shift in the first pass (SVQB: Gram eigenvalues above 1e-14 * max;
 * host, synchronises). */
arr_status orthonormalize(arr_ctx *c, double *X, int64_t ldx, int32_t ncols, int32_t *rank);

/* Augmented Rayleigh-Ritz (Alg. ARR P:531-541 with Alg. RR) on
 * span{X, AX, ..., A^p X}, built as an orthonormal block-Krylov basis
 * Q = [U_0 .. U_p]: U_0 = orth(X), U_j = orth((I - QQ^T) A U_{j-1}) (block CGS2),
 * H = Q^T A Q (m x m, m = (p+1)w, AQ never stored), H = V Theta V^T on device
 * (cuSOLVER syevd; not on the graded path), Y = Q V[:, 1..w].  On one GPU H's
 * block columns 0..p-1 are the first CGS pass's coefficients, block column p
 * keeps its block-tridiagonal rows (R22), its block (p-1, p) is R^T
 * with R the CholeskyQR factor of the last augmentation block (R23; the Gram
 * when that block needed SVQB or re-projection) and block (p, p) is a
 * symmetric-result Gram. 
 * X: n x w input (not modified unless Y == X).  Y: n x w output (the w leading
 * Ritz vectors; may equal X; may be NULL to skip forming them).
 * ritz_host: host [(p+1)w] Ritz values, descending.  rank: host, numerical
 * rank of the basis (min over its blocks' SVQB ranks, summed). */
arr_status arr_project(arr_ctx *c, const double *X, int64_t ldx, double *Y, int64_t ldy,
                       double *ritz_host, int32_t *rank);
/* Same with an explicit depth p_use (0 = plain RR, Alg. RR), p_use <= p. */
arr_status arr_project_p(arr_ctx *c, int32_t p_use, const double *X, int64_t ldx, double *Y,
                         int64_t ldy, double *ritz_host, int32_t *rank);

/* ---------------------------------------------------------------- A6
 * res_i = ||A y_i - mu_i y_i||_2 / max(1, |mu_i|), i < ncols (Eq. resi,
 * P:1322-1325): one fused SpMM with a per-column shift and column sums of
 * squares; the residual block is never written.  mu_host, res_host: host. */
arr_status residuals(arr_ctx *c, const double *Y, int64_t ldy, const double *mu_host, int32_t ncols,
                     double *res_host);

/* ---------------------------------------------------------------- driver
 * Fixed-parameter ARRABIT-MPM (Alg. Arrabit2 P:1463-1527 with the adaptive
 * lines disabled; R3, R6, R10):
 *   a = Gershgorin lower bound; b = smallest Ritz value of RR(A, X0);
 *   repeat: s = sweeps rule; s x filter_step(normalize);  ARR;  residuals;
 *           stop if max res <= tol;  b = mu_{w+1} (monotone once the residual grew, R3);  X = leading Ritz vectors.
 * X: in = X0 (n x w), out = the k Ritz vectors.  eigval_host/res_host: host [k].
 * Returns ARR_OK also when not converged (info->converged = 0). */
arr_status eig_solve(arr_ctx *c, double *X, int64_t ldx, const arr_solve_opts *opts,
                     double *eigval_host, double *res_host, arr_solve_info *info);

/* Host-buffer convenience entry (the public "e2e" call): copies the CSR and X0
 * (n x w, row-major, ld = w; w >= k, w - k guard columns) from host memory to
 * the device, runs eig_solve on a fresh context, copies the k eigenvalues,
 * residuals and eigenvectors (n x k, row-major, ld = k; evec may be NULL) back.
 * All host pointers; device memory is allocated and freed inside, from the device's
 * default stream-ordered pool, which keeps up to min(this call's footprint, a quarter
 * of the device) cached for the next call (ARRABIT_POOL_KEEP=0: 4 GiB;
 * cudaMemPoolTrimTo on the default pool releases it). */
arr_status eig_solve_host(int64_t n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                          const double *val, int32_t k, int32_t w, int32_t p, int32_t d, const double *X0,
                          const arr_solve_opts *opts, double *eigval, double *res, double *evec,
                          arr_solve_info *info, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* ARRABIT_H */
