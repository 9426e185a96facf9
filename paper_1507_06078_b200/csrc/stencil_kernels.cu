// Stencil-aware fused filter degree for sm_100a ("structured path";
// Survey §8f-4).  Same operation and the same per-row FMA order as the CSR kernels
// of spmm_kernels.cu (Eq. cheby-poly P:377-383 on the map of Eq. rhod P:1225-1232,
// Alg. Arrabit2 line P:1486; the augmentation SpMM of Alg. ARR):
//     Y_{j+1} = alpha (A Y_j - shift Y_j) + beta Y_{j-1} (+ gxa X)
// for a matrix whose pattern lies in the 3x3x3 neighbourhood of an nx x ny x nz grid
// (x fastest; the finite-difference operators the paper's test set comes from,
// P:1624-1627).  eig_set_stencil verifies the CSR pattern on the device and stores A
// as K diagonals (DIA, [n][K], zeros where a neighbour is absent).
//
// Why: the per-degree CSR kernel gathers every neighbour row through L1/L2; for the
// 7- and 27-point operators at w = 282..550 that is 5-21 block-sized passes of
// L2 -> SM traffic per degree, and the L2 (~6300 B/clk chip-wide) saturates before
// HBM does.  Here a CTA owns a Px x Py patch of grid lines and a column panel and
// marches along z: plane z's patch (plus its x/y halo) is copied ONCE into shared
// memory by the bulk-copy engine (cp.async.bulk, mbarrier complete_tx, NS-stage
// ring, one producer warp), and every staged row is used for the three output
// planes z-1, z, z+1 from registers (three rotating accumulators per output).  L2 ->
// SM traffic per degree drops to (box/patch) + 2 blocks.  The terms of each output
// row are still added in ascending column order (plane z-1, then z, then z+1; within
// a plane (dy, dx) ascending): bitwise the CSR kernels' sums.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "internal.cuh"

namespace {

// One CTA per SM: 31 consumer warps (one output vector each per step) + 1 producer warp
template <int NT>
struct StCta {
    static constexpr int THREADS = NT, CONS = NT - 32, MINB = 1;
};
constexpr int kStThreads = 1024;

// work items from the atomic ticket in launches without column sums (ARRABIT_ST_DYN=0: static)
int st_dyn() {
    static const int v = [] { const char *e = getenv("ARRABIT_ST_DYN"); return e ? atoi(e) : 1; }();
    return v;
}
// z-chunks per column of patches under the ticket (ARRABIT_ST_NZC; 0 = automatic)
int st_nzc() {
    static const int v = [] { const char *e = getenv("ARRABIT_ST_NZC"); return e ? atoi(e) : 0; }();
    return v;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ uint64_t pol_of(int kind) {  // 0 evict_normal, 1 evict_last, 2 evict_first
    uint64_t p;
    if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void st_stream(double *p, double2 v, uint64_t pol) {
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
                 "l"(pol)
                 : "memory");
}
// alpha (acc - shift y_i): the same contraction as the CSR kernels' epilogue
__device__ __forceinline__ double epi(double alpha, double acc, double shift, double yi) {
    return alpha * fma(-shift, yi, acc);
}
__device__ __forceinline__ void fma2(double2 &acc, double a, const double2 &x) {
    acc.x = fma(a, x.x, acc.x);
    acc.y = fma(a, x.y, acc.y);
}

// Compile-time stencil shapes.  In-plane positions q are in (dy, dx) ascending order
// (the order of each output's terms within a plane); k(dz, q) is the DIA slot of
// neighbour (dx, dy, dz) = (dx(q), dy(q), dz), -1 if the shape has none.  Slots are
// numbered in ascending column order.  A verified pattern runs on the smallest shape
// containing it (absent neighbours are zero slots: exact no-op FMAs).
//   0: 27-point (full 3x3x3)            1: 7-point (3-D)
//   2: 5-point of a 2-D grid declared (nx, 1, ny): x-neighbours in plane, y = march
//   3: 3-point (1-D)
template <int SH>
struct Shape;
template <>
struct Shape<0> {
    static constexpr int NQ = 9, K = 27, QC = 4;
    static constexpr __host__ __device__ int dy(int q) { return q / 3 - 1; }
    static constexpr __host__ __device__ int dx(int q) { return q % 3 - 1; }
    static constexpr __host__ __device__ int k(int dz, int q) { return (dz + 1) * 9 + q; }
};
template <>
struct Shape<1> {
    static constexpr int NQ = 5, K = 7, QC = 2;
    static constexpr __host__ __device__ int dy(int q) { return q == 0 ? -1 : (q == 4 ? 1 : 0); }
    static constexpr __host__ __device__ int dx(int q) { return q == 1 ? -1 : (q == 3 ? 1 : 0); }
    static constexpr __host__ __device__ int k(int dz, int q) { return dz == 0 ? 1 + q : (q == 2 ? (dz < 0 ? 0 : 6) : -1); }
};
template <>
struct Shape<2> {
    static constexpr int NQ = 3, K = 5, QC = 1;
    static constexpr __host__ __device__ int dy(int) { return 0; }
    static constexpr __host__ __device__ int dx(int q) { return q - 1; }
    static constexpr __host__ __device__ int k(int dz, int q) { return dz == 0 ? 1 + q : (q == 1 ? (dz < 0 ? 0 : 4) : -1); }
};
template <>
struct Shape<3> {
    static constexpr int NQ = 3, K = 3, QC = 1;
    static constexpr __host__ __device__ int dy(int) { return 0; }
    static constexpr __host__ __device__ int dx(int q) { return q - 1; }
    static constexpr __host__ __device__ int k(int dz, int q) { return dz == 0 ? q : -1; }
};
template <int SH>
__host__ __device__ bool shape_needs(int ly, int lx, int hy, int hx, int pye, int pxe) {
    bool need = false;
#pragma unroll
    for (int q = 0; q < Shape<SH>::NQ; ++q) {
        const int oy = ly - hy - Shape<SH>::dy(q), ox = lx - hx - Shape<SH>::dx(q);
        need = need || (oy >= 0 && oy < pye && ox >= 0 && ox < pxe);
    }
    return need;
}
template <int SH>
unsigned shape_mask() {
    unsigned m = 0;
    for (int dz = -1; dz <= 1; ++dz)
        for (int q = 0; q < Shape<SH>::NQ; ++q)
            if (Shape<SH>::k(dz, q) >= 0) m |= 1u << ((dz + 1) * 9 + (Shape<SH>::dy(q) + 1) * 3 + (Shape<SH>::dx(q) + 1));
    return m;
}
template <int SH>
void shape_slots(StencilSlots &sl) {
    for (int b = 0; b < 27; ++b) sl.slot[b] = -1;
    for (int dz = -1; dz <= 1; ++dz)
        for (int q = 0; q < Shape<SH>::NQ; ++q)
            if (Shape<SH>::k(dz, q) >= 0)
                sl.slot[(dz + 1) * 9 + (Shape<SH>::dy(q) + 1) * 3 + (Shape<SH>::dx(q) + 1)] = Shape<SH>::k(dz, q);
    sl.K = Shape<SH>::K;
}

// Work item -> patch / panel / z-chunk (panel fastest: a CTA keeps one panel when
// gridDim.x is a multiple of npan, which makes its column partial sums static).
struct Item {
    int panel, x0, y0, pxe, pye, zc0, zc1;
};
// Order of the work items.  Panel-major (PM): it = ((zc npan + panel) npy + py) npx + px,
// so the G items running together are ~G patches of ONE panel in raster order: the x and y
// halo lines two neighbouring patches both stage are fetched from DRAM once and hit L2 the
// second time (panel-minor waves cover only G / (npx npan) patch rows).  Launches that
// reduce column norms keep the panel-minor order, where a CTA owns one panel and its
// partial sums stay static.
template <bool PM>
__device__ __forceinline__ Item decode_item(const StencilLaunch &P, int64_t it) {
    Item r;
    int px, py, zc;
    if (PM) {
        px = (int)(it % P.npx);
        int64_t q = it / P.npx;
        py = (int)(q % P.npy);
        q /= P.npy;
        r.panel = (int)(q % P.npan);
        zc = (int)(q / P.npan);
    } else {
        r.panel = (int)(it % P.npan);
        int64_t q = it / P.npan;
        px = (int)(q % P.npx);
        q /= P.npx;
        py = (int)(q % P.npy);
        zc = (int)(q / P.npy);
    }
    r.x0 = px * P.Px;
    r.y0 = py * P.Py;
    r.pxe = min(P.Px, P.nx - r.x0);
    r.pye = min(P.Py, P.ny - r.y0);
    r.zc0 = P.z0 + zc * P.zstep;
    r.zc1 = min(P.z1, r.zc0 + P.Lz);
    return r;
}

// Shared memory of one CTA: [full[4] | empty[4] mbarriers | meta[4] (128 B)] [NS stages]
// [val ring], every region 128-byte aligned (TMA destinations):
// stage:    box of Y_j (box_y lines x box_x rows x pwv 16-byte vectors) | Y_{j-1} rows |
//           X rows (Py lines x Px rows each)
// val ring: VS = NS + 2 slots, one plane of the patch's DIA rows (Py lines x Px rows x Kpad)
template <bool HAS_PREV, bool HAS_X>
struct StageLayout {
    uint32_t box, prev, xa, dg, bytes;
    // dg_bytes: the diagonal of the patch's plane (value mode 1), 0 otherwise
    __host__ __device__ StageLayout(int nbox, int nrow_max, int pwv, uint32_t dg_bytes = 0) {
        box = 0;
        prev = (uint32_t)nbox * pwv * 16u;
        xa = prev + (HAS_PREV ? (uint32_t)nrow_max * pwv * 16u : 0u);
        dg = xa + (HAS_X ? (uint32_t)nrow_max * pwv * 16u : 0u);
        bytes = dg + ((dg_bytes + 127u) & ~127u);
    }
};
__host__ __device__ inline uint32_t vdiag_bytes(int Pxe, int Py) { return (uint32_t)Pxe * Py * 8u; }
// one DIA plane of a patch (the TMA box's bytes) and its ring slot (128-byte aligned)
__host__ __device__ inline uint32_t vplane_bytes(int Px, int Py, int Kpad) { return (uint32_t)Px * Py * Kpad * 8u; }
__host__ __device__ inline uint32_t vslot_bytes(int Px, int Py, int Kpad) { return (vplane_bytes(Px, Py, Kpad) + 127u) & ~127u; }

// one 4-D box (columns, x, y, z) of a tensor map global -> shared; coordinates outside the
// grid (x = -1 / nx, y = -1 / ny, columns >= w) are zero-filled and count in complete_tx
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap *map, int c0, int x, int y, int z,
                                       uint32_t bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3, %4, %5}], [%6], %7;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(x), "r"(y), "r"(z), "r"(bar), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap *map, int x, int y, int z, uint32_t bar,
                                       uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
        "%3, %4}], [%5], %6;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar), "l"(pol)
        : "memory");
}

// VM: value mode (StencilState::vmode): 0 the K diagonals staged per plane (ring of NS + 2
// planes: the dz = +1 / 0 / -1 terms of one staged Y_j plane need the DIA rows of planes
// z - 1, z, z + 1); 1 constant off-diagonal coefficients (kernel parameters) and the
// diagonal of plane z staged with the plane's box; 2 all coefficients constant.
template <int SH, bool HAS_PREV, bool SUMSQ, bool HAS_X, int NT, int VM>
__global__ void __launch_bounds__(NT, StCta<NT>::MINB) stencil_kernel(const __grid_constant__ StencilLaunch P) {
    using Sh = Shape<SH>;
    constexpr int kStCons = StCta<NT>::CONS;
    extern __shared__ __align__(128) unsigned char sm_raw[];
    unsigned char *sm = sm_raw + ((128u - (smem_u32(sm_raw) & 127u)) & 127u);  // 128-byte aligned base
    uint64_t *full = reinterpret_cast<uint64_t *>(sm);
    uint64_t *empty = full + 4;
    // meta[b]: the work item whose first step stage b holds (-1: no more items), written by
    // the producer before its arrive on full[b] (release) and read after the wait (acquire)
    volatile int64_t *meta = reinterpret_cast<volatile int64_t *>(sm + 64);
    unsigned char *stages = sm + 128;
    const int tid = threadIdx.x;
    const int NS = P.NS, VS = P.NS + 2;
    const StageLayout<HAS_PREV, HAS_X> SL(P.box_x * P.box_y, P.Px * P.Py, P.pwv,
                                           VM == 1 ? vdiag_bytes(P.Pxe, P.Py) : 0u);
    const uint32_t slot_bytes = VM == 0 ? vslot_bytes(P.Px, P.Py, P.Kpad) : 0u;
    unsigned char *vring = stages + (size_t)NS * SL.bytes;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kStCons / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int64_t G = gridDim.x;
    const int pwv = P.pwv;  // smem row stride in 16-byte vectors (a multiple of 8: 128-byte rows)
    if (tid >= kStCons) {
        // ------------------------------------------------------------ producer warp (lane 0)
        // Per step (plane z of the march; z == nz is a tail step with no plane unless a ghost
        // plane lies above; z == -1 a first step on the ghost plane below) at most five
        // TMA boxes completing on full[b]: the Y_j box of plane z (box_x x box_y rows with the
        // x/y halo), the Y_{j-1} (and X) rows of the outputs of plane z-1, and the DIA rows
        // of plane z+1 (and of plane z on an item's first step).
        if (tid != kStCons) return;
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tm_in)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tm_val)) : "memory");
        const uint64_t pol_keep = pol_of(P.ypol);    // Y_j rows: re-staged by the neighbouring patches
        const uint64_t pol_once = pol_of(P.spol);    // Y_{j-1}, X, DIA: read once
        const uint32_t box_b = (uint32_t)P.box_x * P.box_y * pwv * 16u;
        const uint32_t row_b = (uint32_t)P.Px * P.Py * pwv * 16u;
        const uint32_t val_b = VM == 0 ? vplane_bytes(P.Px, P.Py, P.Kpad) : 0u;
        const uint32_t dg_b = VM == 1 ? vdiag_bytes(P.Pxe, P.Py) : 0u;
        const uint32_t st0 = smem_u32(stages), vr0 = smem_u32(vring), fb0 = smem_u32(full);
        int b = 0;
        uint32_t eph = 0;   // parity of the empty-barrier phase to wait for (from the second round on)
        bool wrapped = false;
        int vs = 0;         // ring slot of the current step's plane
        const bool dyn = !SUMSQ && P.dyn;
        for (int64_t it = blockIdx.x; it < P.nitems;) {
            const Item I = (!SUMSQ && P.pm) ? decode_item<true>(P, it) : decode_item<false>(P, it);
            const int col0 = I.panel * pwv * 2;  // first column of the panel
            const int zs = max(I.zc0 - 1, -P.gz_lo);
            for (int z = zs; z <= I.zc1; ++z) {
                if (wrapped) mbar_wait(empty + b, eph);
                const bool real = z < P.nz + P.gz_hi;
                // the block's plane holding virtual plane z: the ghost planes of a z-slab
                // follow the owned ones (lower first)
                const int zp = z < 0 ? P.nz : (z >= P.nz ? P.nz + P.gz_lo : z);
                const bool fin = z - 1 >= I.zc0;
                // DIA planes to load: z+1 (and z on the first step when z is an output plane)
                const int va0 = (z == zs && z >= I.zc0 && real) ? z : z + 1;
                const int va1 = (z + 1 < I.zc1) ? z + 1 : z;  // inclusive; empty if va1 < va0
                const int nv = (VM == 0 && va1 >= va0) ? va1 - va0 + 1 : 0;
                const uint32_t total = (real ? box_b + dg_b : 0u) +
                                       (fin ? (HAS_PREV ? row_b : 0u) + (HAS_X ? row_b : 0u) : 0u) + (uint32_t)nv * val_b;
                if (z == zs) meta[b] = it;
                const uint32_t fb = fb0 + 8u * b;
                mbar_expect_tx(full + b, total);
                const uint32_t st = st0 + (uint32_t)b * SL.bytes;
                if (real) tma_4d(st + SL.box, &P.tm_in, col0, I.x0 - P.hx, I.y0 - P.hy, zp, fb, pol_keep);
                if (VM == 1 && real) tma_3d(st + SL.dg, &P.tm_val, I.x0, I.y0, z, fb, pol_once);
                if (fin) {
                    if (HAS_PREV) tma_4d(st + SL.prev, &P.tm_prev, col0, I.x0, I.y0, z - 1, fb, pol_once);
                    if (HAS_X) tma_4d(st + SL.xa, &P.tm_xa, col0, I.x0, I.y0, z - 1, fb, pol_once);
                }
                for (int zz = va0; zz < va0 + nv; ++zz) {
                    int sl = vs + (zz - z);
                    if (sl >= VS) sl -= VS;
                    tma_4d(vr0 + (uint32_t)sl * slot_bytes, &P.tm_val, 0, I.x0, I.y0, zz, fb, pol_once);
                }
                if (++b == NS) {
                    b = 0;
                    if (wrapped) eph ^= 1u;
                    wrapped = true;
                }
                if (++vs == VS) vs = 0;
            }
            if (dyn) it = G + (int64_t)atomicAdd(P.sched, 1ull);
            else it += G;
        }
        // end of work: one more stage carrying meta = -1 (no bytes)
        if (wrapped) mbar_wait(empty + b, eph);
        meta[b] = -1;
        mbar_arrive(full + b);
        if (dyn) {
            // the last CTA to finish resets the ticket for the next launch
            __threadfence();
            if (atomicAdd(P.sched + 1, 1ull) == (unsigned long long)G - 1) {
                P.sched[0] = 0;
                P.sched[1] = 0;
                __threadfence();
            }
        }
        return;
    }
    // ---------------------------------------------------------------- consumers
    const uint64_t pols = pol_of(P.opol);
    const int Kp = P.Kpad;
    int b = 0;
    uint32_t fph = 0;   // parity of the full-barrier phase of stage b
    int vs = 0;         // ring slot of the current step's plane (as the producer's)
    double ss0 = 0.0, ss1 = 0.0;
    int panel_of_cta = (int)(blockIdx.x % P.npan);
    const int64_t nxy = (int64_t)P.nx * P.ny;
    for (;;) {
        // the next item is named by the stage of its first step
        mbar_wait(full + b, fph);
        const int64_t it = meta[b];
        if (it < 0) break;
        const Item I = (!SUMSQ && P.pm) ? decode_item<true>(P, it) : decode_item<false>(P, it);
        const int pw = min(pwv, P.wv - I.panel * pwv);
        const int nrow = I.pxe * I.pye;
        const int colv0 = I.panel * pwv;
        const int r = tid / pw;
        const int v = tid - r * pw;
        const bool act = r < nrow;  // (v < pw by construction; the smem rows are pwv wide)
        const int oy = act ? r / I.pxe : 0, ox = act ? r - (r / I.pxe) * I.pxe : 0;
        const int cb = (oy + P.hy) * P.box_x + (ox + P.hx);
        const int rs = oy * P.Px + ox;  // patch row slot (prev / X rows)
        const int64_t rxy = (int64_t)(I.y0 + oy) * P.nx + (I.x0 + ox);
        const uint32_t vo = (uint32_t)rs * Kp * 8u;  // this row's DIA entries within a ring slot
        // smem row of each in-plane position.  Value mode 0: the centre where the neighbour
        // is outside the grid (its DIA slot is zero there); modes 1, 2 (constant coefficients):
        // the neighbour's box row, which the TMA zero-filled (an exact zero term)
        int qoff[Sh::NQ];
#pragma unroll
        for (int q = 0; q < Sh::NQ; ++q) {
            const int gx = I.x0 + ox + Sh::dx(q), gy = I.y0 + oy + Sh::dy(q);
            const bool in = gx >= 0 && gx < P.nx && gy >= 0 && gy < P.ny;
            qoff[q] = ((in || VM != 0) ? cb + Sh::dy(q) * P.box_x + Sh::dx(q) : cb) * pwv + v;
        }
        double *outp = P.Yout + (rxy + (int64_t)I.zc0 * nxy) * P.ld_out + (int64_t)(colv0 + v) * 2;
        // lazy MPM scale of this thread's two columns (SpmmArgs::colscale)
        double2 csc = make_double2(1.0, 1.0);
        if (P.scale_mode != 0 && act) csc = __ldg(reinterpret_cast<const double2 *>(P.colscale) + colv0 + v);
        const double2 bsc = P.scale_mode == 2 ? make_double2(P.beta * csc.x, P.beta * csc.y) : make_double2(P.beta, P.beta);
        const int64_t out_step = nxy * P.ld_out;
        double2 accA = make_double2(0.0, 0.0), accB = make_double2(0.0, 0.0), yiA = make_double2(0.0, 0.0);
        const int zs = max(I.zc0 - 1, -P.gz_lo);
        for (int z = zs; z <= I.zc1; ++z) {
            const bool real = z < P.nz + P.gz_hi;
            const bool fin = z - 1 >= I.zc0;                // out(z-1) completes in this step
            const bool mid = z >= I.zc0 && z < I.zc1;       // out(z) gets its plane-z terms
            const bool nxt = z + 1 < I.zc1;                 // out(z+1) starts with its plane-z terms
            mbar_wait(full + b, fph);
            const unsigned char *st = stages + (size_t)b * SL.bytes;
            const double2 *S = reinterpret_cast<const double2 *>(st + SL.box);
            double2 accC = make_double2(0.0, 0.0), yiB = make_double2(0.0, 0.0);
            double2 yp = make_double2(0.0, 0.0), xa = make_double2(0.0, 0.0);
            if (act) {
                if (real) {
                    const int sp = vs == 0 ? VS - 1 : vs - 1, sn = vs + 1 == VS ? 0 : vs + 1;
                    ARR_CHECK(VM != 0 || vo + (size_t)Sh::K * 8 <= slot_bytes);
                    const double *vp = reinterpret_cast<const double *>(vring + (size_t)sp * slot_bytes + vo);
                    const double *v0 = reinterpret_cast<const double *>(vring + (size_t)vs * slot_bytes + vo);
                    const double *vm = reinterpret_cast<const double *>(vring + (size_t)sn * slot_bytes + vo);
                    // this row's diagonal (value mode 1): plane z, staged with the box
                    const double dgv = VM == 1 ? reinterpret_cast<const double *>(st + SL.dg)[oy * P.Pxe + ox] : 0.0;
                    constexpr int kc = Sh::k(0, Sh::QC);  // the centre (diagonal) slot
                    auto cf = [&](const double *v, int k) -> double {
                        if (VM == 0) return v[k];
                        if (VM == 1 && k == kc) return dgv;
                        return P.coef[k];
                    };
                    // the staged plane's terms: row z-1 gets its dz = +1 terms (fin), row z its
                    // dz = 0 terms (mid), row z+1 its dz = -1 terms (nxt).  Interior steps (all
                    // three) run a branch-free copy; the first and last steps of an item the
                    // predicated one.
                    auto terms = [&](auto F, auto M, auto N) {
#pragma unroll
                        for (int q = 0; q < Sh::NQ; ++q) {
                            ARR_CHECK(qoff[q] >= 0 && qoff[q] < P.box_x * P.box_y * pwv);
                            const double2 y = S[qoff[q]];
                            if (q == Sh::QC) yiB = y;
                            if (Sh::k(1, q) >= 0 && F()) fma2(accA, cf(vp, Sh::k(1, q)), y);
                            if (Sh::k(0, q) >= 0 && M()) fma2(accB, cf(v0, Sh::k(0, q)), y);
                            if (Sh::k(-1, q) >= 0 && N()) fma2(accC, cf(vm, Sh::k(-1, q)), y);
                        }
                    };
                    if (fin && mid && nxt) {
                        terms([] { return true; }, [] { return true; }, [] { return true; });
                    } else {
                        terms([&] { return fin; }, [&] { return mid; }, [&] { return nxt; });
                    }
                }
                if (fin) {
                    ARR_CHECK(rs * pwv + v < P.Px * P.Py * pwv && ox < I.pxe && oy < I.pye);
                    if (HAS_PREV) yp = reinterpret_cast<const double2 *>(st + SL.prev)[rs * pwv + v];
                    if (HAS_X) xa = reinterpret_cast<const double2 *>(st + SL.xa)[rs * pwv + v];
                }
            }
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(empty + b);  // this warp is done with stage b
            if (++b == NS) { b = 0; fph ^= 1u; }
            if (++vs == VS) vs = 0;
            if (fin && act) {
                double2 out;
                out.x = epi(P.alpha, accA.x, P.shift, yiA.x);
                out.y = epi(P.alpha, accA.y, P.shift, yiA.y);
                if (HAS_PREV) {
                    out.x = fma(bsc.x, yp.x, out.x);
                    out.y = fma(bsc.y, yp.y, out.y);
                }
                if (HAS_X) {
                    out.x = fma(P.gxa, xa.x, out.x);
                    out.y = fma(P.gxa, xa.y, out.y);
                }
                if (P.scale_mode == 1) {
                    out.x *= csc.x;
                    out.y *= csc.y;
                }
                if (SUMSQ) {
                    ss0 = fma(out.x, out.x, ss0);
                    ss1 = fma(out.y, out.y, ss1);
                }
                st_stream(outp, out, pols);
            }
            if (fin) outp += out_step;
            accA = accB;
            accB = accC;
            yiA = yiB;
        }
    }
    if (SUMSQ) {
        // fixed-order reduction over the consumer threads of each column of this CTA's
        // panel (every stage has landed: all full barriers were waited on), then one
        // partial row of w doubles per CTA (zeros outside the panel)
        asm volatile("bar.sync 1, %0;" ::"r"(kStCons) : "memory");
        double2 *red = reinterpret_cast<double2 *>(stages);
        red[tid] = make_double2(ss0, ss1);
        asm volatile("bar.sync 1, %0;" ::"r"(kStCons) : "memory");
        const int pw = min(pwv, P.wv - panel_of_cta * pwv);
        for (int c = tid; c < P.wv; c += kStCons) {
            double2 s = make_double2(0.0, 0.0);
            const int lc = c - panel_of_cta * pwv;
            if (lc >= 0 && lc < pw) {
                for (int i = lc; i < kStCons; i += pw) {
                    s.x += red[i].x;
                    s.y += red[i].y;
                }
            }
            double *dst = P.partials + (int64_t)blockIdx.x * P.w + 2 * c;
            dst[0] = s.x;
            if (2 * c + 1 < P.w) dst[1] = s.y;
        }
    }
}

// ---------------------------------------------------------------- setup kernels
__device__ __forceinline__ void decode3(int64_t i, int64_t nx, int64_t ny, int64_t &x, int64_t &y, int64_t &z) {
    x = i % nx;
    const int64_t t = i / nx;
    y = t % ny;
    z = t / ny;
}

// Pattern check: sorted, duplicate-free rows whose columns lie in the 3x3x3
// neighbourhood of the row's grid point; OR of the 27 offset bits present.
// Column j of a z-slab's local matrix -> grid point with a VIRTUAL plane: owned columns
// j < n keep z = j / (nx ny); the ghost planes that follow are plane -1 (below, first
// when present) and plane nz (above).
__device__ __forceinline__ void decode_col(int64_t j, int64_t nx, int64_t ny, int64_t nz, int gz_lo, int64_t &x,
                                           int64_t &y, int64_t &z) {
    decode3(j, nx, ny, x, y, z);
    if (z >= nz) z = (gz_lo && z == nz) ? -1 : nz;
}

__global__ void stencil_check_kernel(const int64_t *__restrict__ rp, const int32_t *__restrict__ col, int64_t n,
                                     int64_t nx, int64_t ny, int64_t nz, int gz_lo, int gz_hi, unsigned *mask,
                                     int *bad) {
    const int64_t ncol = n + (int64_t)(gz_lo + gz_hi) * nx * ny;
    unsigned m = 0;
    int b = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t x, y, z;
        decode3(i, nx, ny, x, y, z);
        int64_t prev = -1;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            const int64_t j = col[p];
            if (j < 0 || j >= ncol) { b = 1; break; }
            int64_t xj, yj, zj;
            decode_col(j, nx, ny, nz, gz_lo, xj, yj, zj);
            const int64_t key = xj + nx * (yj + ny * (zj + 1));  // ascending in the global column order
            if (key <= prev) { b = 1; break; }
            prev = key;
            const int64_t dx = xj - x, dy = yj - y, dz = zj - z;
            if (dx < -1 || dx > 1 || dy < -1 || dy > 1 || dz < -1 || dz > 1) { b = 1; break; }
            m |= 1u << ((dz + 1) * 9 + (dy + 1) * 3 + (dx + 1));
        }
    }
    m = __reduce_or_sync(0xffffffffu, m);
    b = __reduce_or_sync(0xffffffffu, (unsigned)b);
    if ((threadIdx.x & 31) == 0) {
        if (m) atomicOr(mask, m);
        if (b) atomicOr(bad, 1);
    }
}

// DIA values: dia[i*K + slot(bit)] = A_ij (0 where the neighbour is absent)
__global__ void stencil_fill_kernel(const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                                    const double *__restrict__ val, int64_t n, int64_t nx, int64_t ny,
                                    int64_t nz, int gz_lo, StencilSlots sl, double *__restrict__ dia) {
    const int Kp = (sl.K + 1) & ~1;  // rows padded to 16 bytes (bulk copies)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double *row = dia + i * Kp;
        for (int k = 0; k < Kp; ++k) row[k] = 0.0;
        int64_t x, y, z;
        decode3(i, nx, ny, x, y, z);
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
            int64_t xj, yj, zj;
            decode_col(col[p], nx, ny, nz, gz_lo, xj, yj, zj);
            const int bit = (int)((zj - z + 1) * 9 + (yj - y + 1) * 3 + (xj - x + 1));
            row[sl.slot[bit]] = val[p];
        }
    }
}

// Per DIA slot k (blockIdx.y): min and max of the slot's value over the rows whose neighbour
// lies inside the grid (order-preserving int64 keys of the doubles, atomics: deterministic).
__device__ __forceinline__ long long dkey(double v) {
    const long long b = __double_as_longlong(v);
    return b >= 0 ? b : b ^ 0x7fffffffffffffffll;
}
__global__ void stencil_coef_range_kernel(const double *__restrict__ dia, int Kpad, int64_t n, int64_t nx, int64_t ny,
                                          int64_t nz, int gz_lo, int gz_hi, StencilSlots sl, long long *kmin,
                                          long long *kmax) {
    const int k = blockIdx.y;
    int bit = -1;
    for (int b = 0; b < 27; ++b)
        if (sl.slot[b] == k) bit = b;
    if (bit < 0) return;
    const int dz = bit / 9 - 1, dy = (bit / 3) % 3 - 1, dx = bit % 3 - 1;
    long long mn = 0x7fffffffffffffffll, mx = -0x7fffffffffffffffll - 1;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = i % nx, t = i / nx, y = t % ny, z = t / ny;
        if (x + dx < 0 || x + dx >= nx || y + dy < 0 || y + dy >= ny || z + dz < -gz_lo || z + dz >= nz + gz_hi) continue;
        const long long key = dkey(dia[i * Kpad + k]);
        mn = key < mn ? key : mn;
        mx = key > mx ? key : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const long long a = __shfl_xor_sync(0xffffffffu, mn, o), b = __shfl_xor_sync(0xffffffffu, mx, o);
        mn = a < mn ? a : mn;
        mx = b > mx ? b : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(kmin + k, mn);
        atomicMax(kmax + k, mx);
    }
}
__global__ void stencil_diag_extract_kernel(const double *__restrict__ dia, int Kpad, int kc, int64_t n,
                                            double *__restrict__ diag) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        diag[i] = dia[i * Kpad + kc];
}
double key_to_double(long long k) { return __builtin_bit_cast(double, k >= 0 ? k : k ^ 0x7fffffffffffffffll); }

template <int SH, bool HAS_PREV, bool SUMSQ, bool HAS_X, int VM>
int launch_st(arr_ctx *c, StencilLaunch &L) {
    constexpr int NT = kStThreads;
    constexpr int kStCons = StCta<NT>::CONS;
    auto kern = stencil_kernel<SH, HAS_PREV, SUMSQ, HAS_X, NT, VM>;
    const StageLayout<HAS_PREV, HAS_X> SL(L.box_x * L.box_y, L.Px * L.Py, L.pwv, VM == 1 ? vdiag_bytes(L.Pxe, L.Py) : 0u);
    const size_t ring = VM == 0 ? (size_t)(L.NS + 2) * vslot_bytes(L.Px, L.Py, L.Kpad) : 0;
    const size_t smem = 256 + std::max((size_t)L.NS * SL.bytes + ring, (size_t)kStCons * 16);
    static LaunchCache cache;
    const int occ = cached_occupancy(cache, kern, NT, smem);
    int64_t G = (int64_t)c->num_sms * occ;
    static const int pm_env = [] { const char *e = getenv("ARRABIT_ST_ORDER"); return e ? atoi(e) : 1; }();
    // L2 policies (0 evict_normal, 1 evict_last, 2 evict_first) of the Y_j boxes, the once-read
    // operands (Y_{j-1}, X, DIA) and the output stores
    static const int ypol = [] { const char *e = getenv("ARRABIT_ST_YPOL"); return e ? atoi(e) : 1; }();
    static const int spol = [] { const char *e = getenv("ARRABIT_ST_SPOL"); return e ? atoi(e) : 2; }();
    static const int opol = [] { const char *e = getenv("ARRABIT_ST_OPOL"); return e ? atoi(e) : 2; }();
    L.ypol = ypol; L.spol = spol; L.opol = opol;
    static const int verbose = getenv("ARRABIT_ST_VERBOSE") ? 1 : 0;
    if (verbose)
        fprintf(stderr, "stencil plan: shape %d vmode %d w %d Px %d Py %d npan %d pwv %d NS %d Lz %d nzc %d items %lld G %lld smem %zu dyn %d\n",
                SH, VM, L.w, L.Px, L.Py, L.npan, L.pwv, L.NS, L.Lz, L.nzc, (long long)L.nitems, (long long)G, smem,
                SUMSQ ? 0 : st_dyn());
    L.pm = SUMSQ ? 0 : pm_env;
    L.dyn = SUMSQ ? 0 : st_dyn();
    L.sched = c->sched;
    if (!L.pm) G = (G / L.npan) * L.npan;  // panel-minor: each CTA keeps one panel (static column partial sums)
    if (G > L.nitems) G = L.nitems;
    if (G < L.npan) G = L.npan;
    kern<<<(unsigned)G, NT, smem, c->stream>>>(L);
    c->launches++;
    static const char *names[4] = {"stencil_kernel (27-point, DIA, TMA-staged 2.5-D)",
                                   "stencil_kernel (7-point, DIA, TMA-staged 2.5-D)",
                                   "stencil_kernel (2-D 5-point, DIA, TMA-staged 2.5-D)",
                                   "stencil_kernel (1-D 3-point, DIA, TMA-staged 2.5-D)"};
    static const char *names_c[4] = {"stencil_kernel (27-point, constant coefficients, TMA-staged 2.5-D)",
                                     "stencil_kernel (7-point, constant off-diagonals, TMA-staged 2.5-D)",
                                     "stencil_kernel (2-D 5-point, constant off-diagonals, TMA-staged 2.5-D)",
                                     "stencil_kernel (1-D 3-point, constant off-diagonals, TMA-staged 2.5-D)"};
    c->last_kernel = VM == 0 ? names[SH] : names_c[SH];
    return (int)G;
}

template <int SH, int VM>
int dispatch_st_flags(arr_ctx *c, StencilLaunch &L, bool prev, bool ss, bool xa) {
    if (!xa) {
        if (prev && !ss) return launch_st<SH, true, false, false, VM>(c, L);
        if (prev && ss) return launch_st<SH, true, true, false, VM>(c, L);
        if (!prev && !ss) return launch_st<SH, false, false, false, VM>(c, L);
        return launch_st<SH, false, true, false, VM>(c, L);
    }
    if (prev && !ss) return launch_st<SH, true, false, true, VM>(c, L);
    if (prev && ss) return launch_st<SH, true, true, true, VM>(c, L);
    if (!prev && !ss) return launch_st<SH, false, false, true, VM>(c, L);
    return launch_st<SH, false, true, true, VM>(c, L);
}
template <int SH>
int dispatch_st_vm(arr_ctx *c, StencilLaunch &L, bool prev, bool ss, bool xa) {
    switch (c->st.vmode) {
        case 1: return dispatch_st_flags<SH, 1>(c, L, prev, ss, xa);
        case 2: return dispatch_st_flags<SH, 2>(c, L, prev, ss, xa);
        default: return dispatch_st_flags<SH, 0>(c, L, prev, ss, xa);
    }
}

bool al16(const void *p, int64_t ld) { return ((uintptr_t)p % 16 == 0) && (ld % 2 == 0); }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    }();
    return fn;
}

// 4-D fp64 tensor map (columns, x, y, z) over a row-major n x (.) block of an nx x ny x nz
// grid (row = x + nx (y + ny z)), row stride ld doubles; box {box_cols, box_x, box_y, 1};
// out-of-range coordinates are zero-filled.
bool encode_4d(CUtensorMap *m, const double *base, int64_t cols, int64_t ld, int64_t nx, int64_t ny, int64_t nz,
               int box_cols, int box_x, int box_y) {
    auto enc = tensor_encoder();
    if (!enc) return false;
    const cuuint64_t gdim[4] = {(cuuint64_t)cols, (cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t gstride[3] = {(cuuint64_t)ld * 8, (cuuint64_t)(ld * nx) * 8, (cuuint64_t)(ld * nx * ny) * 8};
    const cuuint32_t box[4] = {(cuuint32_t)box_cols, (cuuint32_t)box_x, (cuuint32_t)box_y, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    // no L2 promotion: a box row is a column panel's segment of a grid row; promoting its
    // sectors to 128/256-byte blocks would fetch the neighbouring panel's bytes too
    static const CUtensorMapL2promotion promo = [] {
        const char *e = getenv("ARRABIT_ST_PROMO");
        const int v = e ? atoi(e) : 0;
        return v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                        : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                   : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B : CU_TENSOR_MAP_L2_PROMOTION_NONE;
    }();
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(base), gdim, gstride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
           CUDA_SUCCESS;
}

// 3-D fp64 tensor map (x, y, z) over the diagonal [n] of an nx x ny x nz grid; box
// {box_x, box_y, 1} (box_x even: 16-byte inner box rows; needs nx even for 16-byte strides,
// and box starts at even x: a TMA box row must start 16-byte aligned)
bool encode_diag(CUtensorMap *m, const double *base, int64_t nx, int64_t ny, int64_t nz, int box_x, int box_y) {
    auto enc = tensor_encoder();
    if (!enc || nx % 2 != 0) return false;
    const cuuint64_t gdim[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
    const cuuint64_t gstride[2] = {(cuuint64_t)nx * 8, (cuuint64_t)(nx * ny) * 8};
    const cuuint32_t box[3] = {(cuuint32_t)box_x, (cuuint32_t)box_y, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(base), gdim, gstride, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Host: geometry of one launch (patch, panels, z-chunks, stages) for block width w.
// Cost model: L2 -> SM bytes per output row = staged rows per patch
// row + the streamed operands, plus the DIA row once per panel, divided by the
// useful fraction of the launch (ragged patches, last wave of work items).
bool stencil_plan(const arr_ctx *c, int w, bool has_prev, bool has_x, bool dyn, StencilLaunch &L, int z0, int z1,
                  bool ends_only) {
    const StencilState &S = c->st;
    if (!S.on || w % 2 != 0) return false;
    const int wv = w / 2;
    const int nzr = ends_only ? 2 : z1 - z0;  // output planes of this launch
    if (nzr < 1 || (ends_only && z1 - z0 < 2)) return false;
    const int items_max = kStThreads - 32;  // one output vector per consumer thread (IPT = 2 spills)
    // one CTA per SM at 1024 threads; two at 512 (each up to half the SM's shared memory)
    const size_t smem_max = (size_t)S.smem_optin - 256;
    double best = 1e300;
    bool found = false;
    const int hx = S.hx, hy = S.hy;
    for (int npan = 1; npan <= 16; ++npan) {
        // panel rows of a multiple of 8 vectors (128-byte TMA destinations), <= 256 doubles (TMA box)
        const int pwv = ((wv + npan - 1) / npan + 7) / 8 * 8;
        if (pwv > 128) continue;
        if ((int64_t)(npan - 1) * pwv >= wv) break;  // an empty panel
        for (int Py = 1; Py <= (S.ny > 1 ? 16 : 1); ++Py) {
            for (int Px = 1; Px <= 64; ++Px) {
                const int nrow = Px * Py;
                if ((int64_t)nrow * pwv > items_max) break;
                if (Px > S.nx || Py > S.ny) break;
                // value mode 1 stages the diagonal with x innermost: box starts x0 = k Px must
                // be 16-byte aligned (TMA), so Px even
                if (S.vmode == 1 && Px % 2 != 0) continue;
                const int bx = Px + 2 * hx, by = Py + 2 * hy;
                size_t stage = ((size_t)bx * by + (size_t)nrow * ((has_prev ? 1 : 0) + (has_x ? 1 : 0))) * pwv * 16;
                if (S.vmode == 1) stage += (vdiag_bytes((Px + 1) & ~1, Py) + 127) & ~(size_t)127;
                const size_t slot = S.vmode == 0 ? vslot_bytes(Px, Py, S.Kpad) : 0;
                int NS = 4;
                while (NS >= 2 && (size_t)NS * stage + (size_t)(NS + 2) * slot > smem_max) --NS;
                if (NS < 2) continue;
                const int need = bx * by;  // staged rows: the whole box (one TMA box per plane)
                const int npx = (S.nx + Px - 1) / Px, npy = (S.ny + Py - 1) / Py;
                const double rag = (double)S.nx * S.ny / ((double)npx * Px * npy * Py);
                // z-chunks: enough work items for >= ~12 per CTA, chunks of >= 8 planes
                const int64_t G = (int64_t)c->num_sms;
                // ticket order: whole columns of patches (no z-chunk seams) unless that leaves
                // fewer than ~4 items per CTA; static order: >= ~12 items per CTA
                int nzc = 1;
                if (dyn && st_nzc() > 0) nzc = std::min<int>(st_nzc(), nzr);
                else
                    while ((int64_t)npx * npy * npan * nzc < (dyn ? 4 : 12) * G && nzr / (nzc + 1) >= 8) ++nzc;
                if (ends_only) nzc = 2;  // two single-plane chunks: z0 and z1 - 1
                const int Lz = (nzr + nzc - 1) / nzc;
                nzc = (nzr + Lz - 1) / Lz;
                const int64_t items = (int64_t)npx * npy * npan * nzc;
                const double waves = (double)items / (double)((G / npan) * npan);
                const double tail = waves / std::ceil(waves);
                // planes staged per chunk beyond its Lz outputs (a sub-range of a slab, or a slab
                // with ghost planes, stages the plane below and above as well)
                const int extra = (ends_only || z1 - z0 < S.nz) ? 2 : (nzc > 1 ? 1 : 0) + S.gz_lo + S.gz_hi;
                const double warm = (double)(Lz + extra) / Lz;
                const double rowbytes = 16.0 * wv;
                const double colfill = (double)wv / ((double)npan * pwv);  // OOB columns of the last panel
                const double abytes = S.vmode == 0 ? 8.0 * S.Kpad : (S.vmode == 1 ? 8.0 : 0.0);  // A per row
                double cost = ((double)need / nrow * warm + 1.0 + (has_prev ? 1.0 : 0.0) + (has_x ? 1.0 : 0.0)) * rowbytes +
                              abytes * npan;
                cost /= colfill;
                cost *= 1.0 + 6.0 / nrow;  // fixed per-step cost (barriers, TMA issue) over the outputs of a step
                cost /= rag * tail;
                if (NS == 2) cost *= 1.05;
                if (cost < best) {
                    best = cost;
                    found = true;
                    L.Px = Px; L.Py = Py; L.Lz = Lz;
                    L.npx = npx; L.npy = npy; L.nzc = nzc; L.npan = npan;
                    L.pwv = pwv; L.wv = wv; L.NS = NS;
                    L.box_x = bx; L.box_y = by;
                    L.nitems = items;
                }
            }
        }
    }
    if (!found) return false;
    L.nx = (int)S.nx; L.ny = (int)S.ny; L.nz = (int)S.nz;
    L.gz_lo = S.gz_lo; L.gz_hi = S.gz_hi;
    L.z0 = z0; L.z1 = z1;
    L.zstep = ends_only ? z1 - 1 - z0 : L.Lz;
    L.hx = hx; L.hy = hy;
    L.K = S.K;
    L.Kpad = S.Kpad;
    L.val = S.dia;
    L.vmode = S.vmode;
    L.Pxe = (L.Px + 1) & ~1;
    for (int k = 0; k < 27; ++k) L.coef[k] = S.coef[k];
    L.w = w;
    return true;
}

// Fused SpMM through the stencil path; -1 when it does not apply to this launch.
int launch_spmm_stencil(arr_ctx *c, const SpmmArgs &a, int z0, int z1, bool ends_only) {
    if (!c->st.on || a.colshift || a.n != c->A.n || a.w % 2 != 0) return -1;
    if (z1 < 0) z1 = (int)c->st.nz;
    if (z0 < 0 || z1 > c->st.nz || z0 >= z1) return -1;
    if (!al16(a.Yin, a.ld_in) || !a.Yout || !al16(a.Yout, a.ld_out)) return -1;
    if (a.Yprev && !al16(a.Yprev, a.ld_prev)) return -1;
    if (a.Xa && !al16(a.Xa, a.ld_xa)) return -1;
    StencilLaunch L{};
    if (!stencil_plan(c, a.w, a.Yprev != nullptr, a.Xa != nullptr, !a.partials && st_dyn(), L, z0, z1, ends_only)) return -1;
    L.Yin = a.Yin; L.ld_in = a.ld_in;
    L.Yprev = a.Yprev; L.ld_prev = a.ld_prev;
    L.Yout = a.Yout; L.ld_out = a.ld_out;
    L.Xa = a.Xa; L.ld_xa = a.ld_xa;
    L.alpha = a.alpha; L.shift = a.shift; L.beta = a.beta; L.gxa = a.gxa;
    L.colscale = a.colscale; L.scale_mode = a.colscale ? a.scale_mode : 0;
    L.partials = a.partials;
    const StencilState &S = c->st;
    if (!encode_4d(&L.tm_in, a.Yin, a.w, a.ld_in, S.nx, S.ny, S.nz + S.gz_lo + S.gz_hi, 2 * L.pwv, L.box_x, L.box_y) ||
        (S.vmode == 0 && !encode_4d(&L.tm_val, S.dia, S.Kpad, S.Kpad, S.nx, S.ny, S.nz, S.Kpad, L.Px, L.Py)) ||
        (S.vmode == 1 && !encode_diag(&L.tm_val, S.dia, S.nx, S.ny, S.nz, L.Pxe, L.Py)) ||
        (a.Yprev && !encode_4d(&L.tm_prev, a.Yprev, a.w, a.ld_prev, S.nx, S.ny, S.nz, 2 * L.pwv, L.Px, L.Py)) ||
        (a.Xa && !encode_4d(&L.tm_xa, a.Xa, a.w, a.ld_xa, S.nx, S.ny, S.nz, 2 * L.pwv, L.Px, L.Py)))
        return -1;
    const bool prev = a.Yprev != nullptr, ss = a.partials != nullptr, xa = a.Xa != nullptr;
    switch (c->st.shape) {
        case 0: return dispatch_st_vm<0>(c, L, prev, ss, xa);
        case 1: return dispatch_st_vm<1>(c, L, prev, ss, xa);
        case 2: return dispatch_st_vm<2>(c, L, prev, ss, xa);
        case 3: return dispatch_st_vm<3>(c, L, prev, ss, xa);
    }
    return -1;
}

// Verify the pattern and build the DIA values (eig_set_stencil).
arr_status stencil_setup(arr_ctx *c, int64_t nx, int64_t ny, int64_t nz, int gz_lo, int gz_hi) {
    StencilState &S = c->st;
    if (S.dia) {
        cudaFreeAsync(S.dia, c->stream);
        S.dia = nullptr;
    }
    S.on = false;
    if (nx == 0 && ny == 0 && nz == 0) return ARR_OK;
    if (nx < 1 || ny < 1 || nz < 1 || nx * ny * nz != c->A.n) return ARR_EINVAL;
    unsigned *mask = reinterpret_cast<unsigned *>(c->dinfo + 60);
    int *bad = c->dinfo + 61;
    cudaMemsetAsync(c->dinfo + 60, 0, 2 * sizeof(int), c->stream);
    int64_t blocks = (c->A.n + 255) / 256;
    if (blocks > (int64_t)c->num_sms * 8) blocks = (int64_t)c->num_sms * 8;
    stencil_check_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(c->A.row_ptr, c->A.col_idx, c->A.n, nx, ny, nz, gz_lo,
                                                                   gz_hi, mask, bad);
    c->launches++;
    if (cudaMemcpyAsync(c->h_istage, c->dinfo + 60, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(c->stream) != cudaSuccess)
        return ARR_ECUDA;
    const unsigned m = (unsigned)c->h_istage[0];
    if (c->h_istage[1] || m == 0) return ARR_EINVAL;
    // the smallest compiled shape whose neighbour set contains the pattern (its slots are
    // in ascending column order; absent neighbours stay zero)
    StencilSlots sl{};
    int shape = -1;
    if ((m & ~shape_mask<3>()) == 0) { shape = 3; shape_slots<3>(sl); }
    else if ((m & ~shape_mask<2>()) == 0) { shape = 2; shape_slots<2>(sl); }
    else if ((m & ~shape_mask<1>()) == 0) { shape = 1; shape_slots<1>(sl); }
    else { shape = 0; shape_slots<0>(sl); }
    const int K = sl.K;
    S.shape = shape;
    S.hx = 1;
    S.hy = (shape <= 1 && ny > 1) ? 1 : 0;
    void *dia = nullptr;
    const int Kpad = (K + 1) & ~1;
    if (cudaMallocAsync(&dia, sizeof(double) * (size_t)c->A.n * Kpad, c->stream) != cudaSuccess) {
        cudaGetLastError();
        return ARR_ENOMEM;
    }
    stencil_fill_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(c->A.row_ptr, c->A.col_idx, c->A.val, c->A.n, nx, ny,
                                                                  nz, gz_lo, sl, (double *)dia);
    c->launches++;
    if (cudaGetLastError() != cudaSuccess) return ARR_ECUDA;
    // Constant coefficients (finite-difference operators): every slot's value the same on all
    // rows whose neighbour is in the grid.  Then only the diagonal (vmode 1), or nothing
    // (vmode 2), is read per row; ARRABIT_ST_VMODE caps the mode (0: always the K diagonals).
    S.vmode = 0;
    static const int vcap = [] { const char *e = getenv("ARRABIT_ST_VMODE"); return e ? atoi(e) : 2; }();
    if (vcap > 0) {
        long long *keys = nullptr;
        if (cudaMallocAsync((void **)&keys, sizeof(long long) * 54, c->stream) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeAsync(dia, c->stream);
            return ARR_ENOMEM;
        }
        std::vector<long long> init(54);
        for (int k = 0; k < 27; ++k) { init[k] = 0x7fffffffffffffffll; init[27 + k] = -0x7fffffffffffffffll - 1; }
        cudaMemcpyAsync(keys, init.data(), sizeof(long long) * 54, cudaMemcpyHostToDevice, c->stream);
        stencil_coef_range_kernel<<<dim3((unsigned)blocks, K), 256, 0, c->stream>>>((const double *)dia, Kpad, c->A.n, nx,
                                                                                    ny, nz, gz_lo, gz_hi, sl, keys,
                                                                                    keys + 27);
        c->launches++;
        std::vector<long long> h(54);
        if (cudaMemcpyAsync(h.data(), keys, sizeof(long long) * 54, cudaMemcpyDeviceToHost, c->stream) != cudaSuccess ||
            cudaStreamSynchronize(c->stream) != cudaSuccess) {
            cudaFreeAsync(keys, c->stream);
            cudaFreeAsync(dia, c->stream);
            return ARR_ECUDA;
        }
        cudaFreeAsync(keys, c->stream);
        int kc = -1;
        for (int b = 0; b < 27; ++b)
            if (b == 13) kc = sl.slot[b];  // (0, 0, 0): the diagonal
        bool off_const = true, diag_const = true;
        for (int k = 0; k < K; ++k) {
            const bool present = h[k] <= h[27 + k];
            const bool cst = !present || h[k] == h[27 + k];
            S.coef[k] = present ? key_to_double(h[k]) : 0.0;
            if (k == kc) diag_const = cst;
            else off_const = off_const && cst;
        }
        if (off_const && diag_const && vcap >= 2) {
            S.vmode = 2;
        } else if (off_const && kc >= 0 && nx % 2 == 0) {
            double *diag = nullptr;
            if (cudaMallocAsync((void **)&diag, sizeof(double) * (size_t)c->A.n, c->stream) != cudaSuccess) {
                cudaGetLastError();
            } else {
                stencil_diag_extract_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>((const double *)dia, Kpad, kc, c->A.n,
                                                                                   diag);
                c->launches++;
                cudaFreeAsync(dia, c->stream);
                dia = diag;
                S.vmode = 1;
            }
        }
        if (S.vmode == 2) {
            cudaFreeAsync(dia, c->stream);
            dia = nullptr;
        }
    }
    S.dia = (double *)dia;
    S.nx = nx; S.ny = ny; S.nz = nz;
    S.gz_lo = gz_lo; S.gz_hi = gz_hi;
    S.K = K;
    S.Kpad = Kpad;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    S.smem_optin = optin > 0 ? optin : 227 * 1024;
    S.on = true;
    return ARR_OK;
}

void stencil_release(arr_ctx *c) {
    if (c->st.dia) cudaFreeAsync(c->st.dia, c->stream);
    c->st.dia = nullptr;
    c->st.on = false;
}
