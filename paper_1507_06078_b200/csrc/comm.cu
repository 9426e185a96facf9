// Multi-GPU exchange of the hot path: A is
// row-partitioned, each rank owns a contiguous row block of A and the same rows
// of every n x w block, with the ghost rows its SpMM gathers appended after the
// owned rows.  Before every SpMM the ghost rows of the gathered operand are
// exchanged (halo for stencils; nearly an all-gather for irregular sparsity);
// after every Gram / column-norm partial the w x w (m x m) result is summed
// over ranks.  Two transports implement the same four operations:
//   - NCCL (one process per GPU, NVLink 5 / NVSwitch): grouped ncclSend/ncclRecv
//     on a side stream, overlapped with the SpMM of the interior rows;
//     ncclAllReduce / ncclBroadcast on the context stream.
//   - an in-process group (one host thread per rank, any devices the process
//     can address): the same data movement done with cudaMemcpyAsync and
//     fixed-order reduction kernels, synchronised with host barriers and
//     stream-event waits (no kernel ever waits on another).  It exists so the
//     distributed driver can be tested on one GPU.
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "internal.cuh"

// ---------------------------------------------------------------- communicator
struct LocalSlot {
    const double *ptr = nullptr;        // published buffer (allreduce / bcast source)
    std::vector<const double *> src;    // halo: source of the rows destined to peer index q
    std::vector<int64_t> offs;          // column split: offsets of the pieces for each rank
    cudaEvent_t ready = nullptr, done = nullptr;
    const arr_ctx *ctx = nullptr;       // the context currently attached (peers, offsets)
};

struct LocalGroup {
    int size = 0;
    int refs = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool broken = false;
    std::vector<LocalSlot> slot;

    // generation barrier; false on timeout (a rank failed: the group is broken)
    bool barrier() {
        std::unique_lock<std::mutex> lk(m);
        if (broken) return false;
        const uint64_t g = gen;
        if (++arrived == size) {
            arrived = 0;
            ++gen;
            cv.notify_all();
            return true;
        }
        if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g || broken; }) || broken) {
            broken = true;
            cv.notify_all();
            return false;
        }
        return true;
    }
};

struct arr_comm {
    int rank = 0, size = 1;
    int kind = 0;  // 0 = NCCL, 1 = in-process group
    ncclComm_t nccl = nullptr;
    LocalGroup *group = nullptr;
};

namespace {

// ---------------------------------------------------------------- kernels
// out[q*ld_out + c] = src[rows[q]*ld_in + c]  (gather of the rows to send)
__global__ void pack_rows_kernel(const double *__restrict__ src, int64_t ld_in, const int32_t *__restrict__ rows,
                                 int64_t nrows, int ncols, double *__restrict__ out, int64_t ld_out) {
    const int64_t total = nrows * (int64_t)ncols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = t / ncols;
        const int cc = (int)(t - q * ncols);
        out[q * ld_out + cc] = src[(int64_t)rows[q] * ld_in + cc];
    }
}

// dst[r*ld_dst + c] = src[r*ld_src + c]
__global__ void copy2d_kernel(const double *__restrict__ src, int64_t ld_src, double *__restrict__ dst,
                              int64_t ld_dst, int64_t nrows, int ncols) {
    const int64_t total = nrows * (int64_t)ncols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / ncols;
        const int cc = (int)(t - r * ncols);
        dst[r * ld_dst + cc] = src[r * ld_src + cc];
    }
}

constexpr int kMaxRanks = 64;
struct PtrTable { const double *p[kMaxRanks]; };

// out[i] = op over ranks r = 0..size-1 (in rank order) of in[r][i]
__global__ void reduce_ranks_kernel(PtrTable in, int size, size_t count, int op, double *__restrict__ out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        double s = in.p[0][i];
        for (int r = 1; r < size; ++r) {
            const double x = in.p[r][i];
            s = op == 0 ? s + x : (op == 1 ? fmin(s, x) : fmax(s, x));
        }
        out[i] = s;
    }
}

unsigned grid_for(const arr_ctx *c, int64_t work) {
    int64_t b = (work + 255) / 256;
    const int64_t cap = (int64_t)c->num_sms * 8;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (unsigned)b;
}

arr_status cfail(arr_ctx *c, arr_status code, const std::string &msg) {
    c->err = msg;
    if (code == ARR_ECUDA || code == ARR_ENCCL) c->poisoned = code;
    return code;
}

#define CT(expr)                                                                                          \
    do {                                                                                                  \
        cudaError_t e_ = (expr);                                                                          \
        if (e_ != cudaSuccess) return cfail(c, ARR_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)
#define NT(expr)                                                                                          \
    do {                                                                                                  \
        ncclResult_t r_ = (expr);                                                                         \
        if (r_ != ncclSuccess) return cfail(c, ARR_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
    } while (0)
#define BARRIER(g)                                                                                        \
    do {                                                                                                  \
        if (!(g)->barrier()) return cfail(c, ARR_ENCCL, "in-process group: barrier timed out (a rank failed)"); \
    } while (0)

inline bool multi(const arr_ctx *c) { return c->nranks > 1; }

}  // namespace

// ---------------------------------------------------------------- collectives
arr_status comm_allreduce(arr_ctx *c, double *buf, size_t count, int op) {
    if (!multi(c) || count == 0) return ARR_OK;
    arr_comm *m = c->comm;
    if (m->kind == 0) {
        const ncclRedOp_t o = op == 0 ? ncclSum : (op == 1 ? ncclMin : ncclMax);
        NT(ncclAllReduce(buf, buf, count, ncclFloat64, o, m->nccl, c->stream));
        return ARR_OK;
    }
    LocalGroup *g = m->group;
    if (count > c->stage_elems) return cfail(c, ARR_EINVAL, "allreduce larger than the staging buffer");
    LocalSlot &me = g->slot[m->rank];
    me.ptr = buf;
    CT(cudaEventRecord(me.ready, c->stream));
    BARRIER(g);
    PtrTable t{};
    for (int r = 0; r < g->size; ++r) {
        if (r != m->rank) CT(cudaStreamWaitEvent(c->stream, g->slot[r].ready, 0));
        t.p[r] = g->slot[r].ptr;
    }
    reduce_ranks_kernel<<<grid_for(c, (int64_t)count), 256, 0, c->stream>>>(t, g->size, count, op, c->stage);
    c->launches++;
    CT(cudaGetLastError());
    CT(cudaEventRecord(me.done, c->stream));
    BARRIER(g);
    for (int r = 0; r < g->size; ++r)
        if (r != m->rank) CT(cudaStreamWaitEvent(c->stream, g->slot[r].done, 0));  // peers finished reading buf
    CT(cudaMemcpyAsync(buf, c->stage, sizeof(double) * count, cudaMemcpyDeviceToDevice, c->stream));
    BARRIER(g);  // every rank has queued its wait on our `done` before it is re-recorded
    return ARR_OK;
}

arr_status comm_bcast(arr_ctx *c, double *buf, size_t count, int root) {
    if (!multi(c) || count == 0) return ARR_OK;
    arr_comm *m = c->comm;
    if (m->kind == 0) {
        NT(ncclBroadcast(buf, buf, count, ncclFloat64, root, m->nccl, c->stream));
        return ARR_OK;
    }
    LocalGroup *g = m->group;
    LocalSlot &me = g->slot[m->rank];
    me.ptr = buf;
    CT(cudaEventRecord(me.ready, c->stream));
    BARRIER(g);
    if (m->rank != root) {
        CT(cudaStreamWaitEvent(c->stream, g->slot[root].ready, 0));
        CT(cudaMemcpyAsync(buf, g->slot[root].ptr, sizeof(double) * count, cudaMemcpyDeviceToDevice, c->stream));
    }
    CT(cudaEventRecord(me.done, c->stream));
    BARRIER(g);
    if (m->rank == root)
        for (int r = 0; r < g->size; ++r)
            if (r != root) CT(cudaStreamWaitEvent(c->stream, g->slot[r].done, 0));
    BARRIER(g);
    return ARR_OK;
}

// Start the exchange of the ghost rows of Y (ncols columns, leading dimension
// ld): the rows this rank owns and a peer references are sent, the peer's rows
// this rank references land in Y rows [n_own + recv_off[q], ...).  Rows are sent
// straight from Y when they are contiguous and ld is the packed width, else they
// are packed first; they are received straight into Y when ld is the packed
// width, else into the receive buffer (unpacked by comm_halo_end).
arr_status comm_halo_begin(arr_ctx *c, const double *Y, int64_t ld, int ncols) {
    if (!multi(c)) return ARR_OK;
    DistPlan &P = c->plan;
    arr_comm *m = c->comm;
    const int np = (int)P.peer.size();
    const int64_t ldp = (ncols + 1) & ~1;
    const bool direct = (ld == ldp);
    P.cur_direct = direct;
    P.cur_ncols = ncols;
    P.cur_ld = ld;
    bool need_pack = false;
    for (int q = 0; q < np; ++q) need_pack = need_pack || !(direct && P.send_contig[q]);
    if (need_pack && P.send_off[np] > 0) {
        pack_rows_kernel<<<grid_for(c, P.send_off[np] * ncols), 256, 0, c->stream>>>(Y, ld, P.send_rows_dev,
                                                                                      P.send_off[np], ncols,
                                                                                      P.sendbuf, ldp);
        c->launches++;
        CT(cudaGetLastError());
    }
    std::vector<const double *> src(np);
    std::vector<double *> dst(np);
    for (int q = 0; q < np; ++q) {
        src[q] = (direct && P.send_contig[q]) ? Y + P.send_first[q] * ld : P.sendbuf + P.send_off[q] * ldp;
        dst[q] = direct ? const_cast<double *>(Y) + (c->A.n + P.recv_off[q]) * ld : P.recvbuf + P.recv_off[q] * ldp;
    }
    CT(cudaEventRecord(P.ev_ready, c->stream));
    if (m->kind == 0) {
        CT(cudaStreamWaitEvent(P.comm_stream, P.ev_ready, 0));
        NT(ncclGroupStart());
        for (int q = 0; q < np; ++q) {
            const size_t ns = (size_t)(P.send_off[q + 1] - P.send_off[q]) * ldp;
            const size_t nr = (size_t)(P.recv_off[q + 1] - P.recv_off[q]) * ldp;
            if (ns) NT(ncclSend(src[q], ns, ncclFloat64, P.peer[q], m->nccl, P.comm_stream));
            if (nr) NT(ncclRecv(dst[q], nr, ncclFloat64, P.peer[q], m->nccl, P.comm_stream));
        }
        NT(ncclGroupEnd());
        CT(cudaEventRecord(P.ev_done, P.comm_stream));
        return ARR_OK;
    }
    // in-process group: publish the sources, then pull every peer's rows
    LocalGroup *g = m->group;
    LocalSlot &me = g->slot[m->rank];
    me.src = src;
    CT(cudaEventRecord(me.ready, c->stream));
    BARRIER(g);
    CT(cudaStreamWaitEvent(P.comm_stream, P.ev_ready, 0));
    for (int q = 0; q < np; ++q) {
        const size_t nr = (size_t)(P.recv_off[q + 1] - P.recv_off[q]) * ldp;
        if (!nr) continue;
        const LocalSlot &ps = g->slot[P.peer[q]];
        const DistPlan &PP = ps.ctx->plan;
        int qi = -1;  // my index in the peer's list
        for (int t = 0; t < (int)PP.peer.size(); ++t)
            if (PP.peer[t] == m->rank) qi = t;
        if (qi < 0 || (size_t)(PP.send_off[qi + 1] - PP.send_off[qi]) * ldp != nr)
            return cfail(c, ARR_EINVAL, "halo plans of two ranks disagree");
        CT(cudaStreamWaitEvent(P.comm_stream, ps.ready, 0));
        CT(cudaMemcpyAsync(dst[q], ps.src[qi], sizeof(double) * nr, cudaMemcpyDeviceToDevice, P.comm_stream));
    }
    CT(cudaEventRecord(P.ev_done, P.comm_stream));
    CT(cudaEventRecord(me.done, P.comm_stream));
    return ARR_OK;
}

// Make the context stream wait for the ghost rows of Y (and unpack them).
arr_status comm_halo_end(arr_ctx *c, double *Y) {
    if (!multi(c)) return ARR_OK;
    DistPlan &P = c->plan;
    arr_comm *m = c->comm;
    if (m->kind == 1) {
        LocalGroup *g = m->group;
        BARRIER(g);  // every peer has queued its pulls of our rows
        for (int q = 0; q < (int)P.peer.size(); ++q) CT(cudaStreamWaitEvent(c->stream, g->slot[P.peer[q]].done, 0));
    }
    CT(cudaStreamWaitEvent(c->stream, P.ev_done, 0));
    if (!P.cur_direct && P.n_ghost > 0) {
        const int64_t ldp = (P.cur_ncols + 1) & ~1;
        copy2d_kernel<<<grid_for(c, P.n_ghost * P.cur_ncols), 256, 0, c->stream>>>(
            P.recvbuf, ldp, Y + c->A.n * P.cur_ld, P.cur_ld, P.n_ghost, P.cur_ncols);
        c->launches++;
        CT(cudaGetLastError());
    }
    if (m->kind == 1) BARRIER(m->group);  // all waits on our events are queued before they are re-recorded
    return ARR_OK;
}

// ---------------------------------------------------------------- column <-> row transposes
// Column-partitioned mode (Survey §8f-3): rank r holds columns [cb[r], cb[r+1]) of every
// n x w block (all rows; "column layout") and, for the ARR projection, rows
// [rb[r], rb[r+1]) of all w columns ("row layout", the row context's owned rows).
// col2row moves the column layout to the row layout, row2col back: one all-to-all each,
// through packed buffers whose row stride is the (even) sender width.
namespace {
inline int64_t ev(int64_t x) { return (x + 1) & ~int64_t(1); }
}  // namespace

arr_status comm_transpose(arr_ctx *c, const ColSplit &S, int dir, const double *src, int64_t lds, double *dst,
                          int64_t ldd) {
    arr_comm *m = c->comm;
    const int R = m->rank, G = m->size;
    const int64_t wr = S.cb[R + 1] - S.cb[R], nr = S.rb[R + 1] - S.rb[R];
    // send piece for peer q and where it lands on q (row layout: rows of q x my columns;
    // column layout: my rows x q's columns), packed with row stride ev(width)
    std::vector<int64_t> soff(G + 1, 0), roff(G + 1, 0);
    for (int q = 0; q < G; ++q) {
        const int64_t nq = S.rb[q + 1] - S.rb[q], wq = S.cb[q + 1] - S.cb[q];
        soff[q + 1] = soff[q] + (dir == 0 ? nq * ev(wr) : nr * ev(wq));
        roff[q + 1] = roff[q] + (dir == 0 ? nr * ev(wq) : nq * ev(wr));
    }
    if (soff[G] > (int64_t)S.buf_elems || roff[G] > (int64_t)S.buf_elems)
        return cfail(c, ARR_EINVAL, "column split: transpose buffer too small");
    // pack
    for (int q = 0; q < G; ++q) {
        const int64_t nq = S.rb[q + 1] - S.rb[q], wq = S.cb[q + 1] - S.cb[q];
        if (dir == 0) {  // my columns, rows of q
            if (nq && wr)
                copy2d_kernel<<<grid_for(c, nq * wr), 256, 0, c->stream>>>(src + S.rb[q] * lds, lds, S.sendbuf + soff[q],
                                                                           ev(wr), nq, (int)wr);
        } else {  // my rows, columns of q
            if (nr && wq)
                copy2d_kernel<<<grid_for(c, nr * wq), 256, 0, c->stream>>>(src + S.cb[q], lds, S.sendbuf + soff[q],
                                                                           ev(wq), nr, (int)wq);
        }
        c->launches++;
    }
    CT(cudaGetLastError());
    if (m->kind == 0) {
        if (roff[R + 1] > roff[R])  // own piece: a device copy
            CT(cudaMemcpyAsync(S.recvbuf + roff[R], S.sendbuf + soff[R], sizeof(double) * (roff[R + 1] - roff[R]),
                               cudaMemcpyDeviceToDevice, c->stream));
        NT(ncclGroupStart());
        for (int q = 0; q < G; ++q) {
            if (q == R) continue;
            if (soff[q + 1] > soff[q]) NT(ncclSend(S.sendbuf + soff[q], soff[q + 1] - soff[q], ncclFloat64, q, m->nccl, c->stream));
            if (roff[q + 1] > roff[q]) NT(ncclRecv(S.recvbuf + roff[q], roff[q + 1] - roff[q], ncclFloat64, q, m->nccl, c->stream));
        }
        NT(ncclGroupEnd());
    } else {
        LocalGroup *g = m->group;
        LocalSlot &me = g->slot[R];
        me.src.assign(1, S.sendbuf);
        me.offs = soff;
        CT(cudaEventRecord(me.ready, c->stream));
        BARRIER(g);
        for (int q = 0; q < G; ++q) {
            const LocalSlot &ps = g->slot[q];
            const int64_t cnt = roff[q + 1] - roff[q];
            if (!cnt) continue;
            if ((int64_t)ps.offs.size() != G + 1 || ps.offs[R + 1] - ps.offs[R] != cnt)
                return cfail(c, ARR_EINVAL, "column split: the ranks' transpose plans disagree");
            if (q != R) CT(cudaStreamWaitEvent(c->stream, ps.ready, 0));
            CT(cudaMemcpyAsync(S.recvbuf + roff[q], ps.src[0] + ps.offs[R], sizeof(double) * cnt,
                               cudaMemcpyDeviceToDevice, c->stream));
        }
        CT(cudaEventRecord(me.done, c->stream));
        BARRIER(g);
        for (int q = 0; q < G; ++q)
            if (q != R) CT(cudaStreamWaitEvent(c->stream, g->slot[q].done, 0));  // peers finished reading our sendbuf
        BARRIER(g);
    }
    // unpack
    for (int q = 0; q < G; ++q) {
        const int64_t nq = S.rb[q + 1] - S.rb[q], wq = S.cb[q + 1] - S.cb[q];
        if (dir == 0) {  // rows of mine x columns of q -> row layout
            if (nr && wq)
                copy2d_kernel<<<grid_for(c, nr * wq), 256, 0, c->stream>>>(S.recvbuf + roff[q], ev(wq), dst + S.cb[q], ldd,
                                                                           nr, (int)wq);
        } else {  // rows of q x my columns -> column layout
            if (nq && wr)
                copy2d_kernel<<<grid_for(c, nq * wr), 256, 0, c->stream>>>(S.recvbuf + roff[q], ev(wr), dst + S.rb[q] * ldd,
                                                                           ldd, nq, (int)wr);
        }
        c->launches++;
    }
    CT(cudaGetLastError());
    return ARR_OK;
}

// ---------------------------------------------------------------- plan setup
arr_status comm_setup_plan(arr_ctx *c, const arr_dist *d, arr_comm *m) {
    DistPlan &P = c->plan;
    c->comm = m;
    c->nranks = m->size;
    P.n_global = d->n_global;
    P.row_begin = d->row_begin;
    P.n_ghost = d->n_ghost;
    const int np = d->npeers;
    if (np < 0 || (np > 0 && (!d->peer || !d->send_off || !d->recv_off)) || d->n_ghost < 0)
        return cfail(c, ARR_EINVAL, "dist: bad peer lists");
    P.peer.assign(d->peer, d->peer + np);
    P.send_off.assign(d->send_off, d->send_off + np + 1);
    P.recv_off.assign(d->recv_off, d->recv_off + np + 1);
    if (np == 0) { P.send_off = {0}; P.recv_off = {0}; }
    if (P.recv_off[np] != P.n_ghost) return cfail(c, ARR_EINVAL, "dist: recv_off[npeers] != n_ghost");
    for (int q = 0; q < np; ++q) {
        if (P.peer[q] < 0 || P.peer[q] >= m->size || P.peer[q] == m->rank)
            return cfail(c, ARR_EINVAL, "dist: bad peer rank");
        if (P.send_off[q + 1] < P.send_off[q] || P.recv_off[q + 1] < P.recv_off[q])
            return cfail(c, ARR_EINVAL, "dist: offsets not nondecreasing");
    }
    const int64_t ns = P.send_off[np];
    P.send_contig.assign(np, 0);
    P.send_first.assign(np, 0);
    for (int q = 0; q < np; ++q) {
        bool contig = true;
        for (int64_t t = P.send_off[q]; t < P.send_off[q + 1]; ++t) {
            const int32_t r = d->send_rows[t];
            if (r < 0 || r >= c->A.n) return cfail(c, ARR_EINVAL, "dist: send row out of range");
            if (t > P.send_off[q] && r != d->send_rows[t - 1] + 1) contig = false;
        }
        P.send_contig[q] = contig;
        P.send_first[q] = P.send_off[q + 1] > P.send_off[q] ? d->send_rows[P.send_off[q]] : 0;
    }
    const int64_t ldp = ((int64_t)c->w + 1) & ~int64_t(1);
    CT(cudaMalloc(&P.send_rows_dev, sizeof(int32_t) * (size_t)std::max<int64_t>(ns, 1)));
    if (ns) CT(cudaMemcpy(P.send_rows_dev, d->send_rows, sizeof(int32_t) * ns, cudaMemcpyHostToDevice));
    CT(cudaMalloc(&P.sendbuf, sizeof(double) * (size_t)std::max<int64_t>(ns * ldp, 1)));
    CT(cudaMalloc(&P.recvbuf, sizeof(double) * (size_t)std::max<int64_t>(P.n_ghost * ldp, 1)));
    // interior / boundary row tiles (processing order; together an exact cover of the owned rows)
    auto up = [&](const int64_t *r0, const int32_t *ln, int64_t nt, int64_t **dr0, int32_t **dln) -> arr_status {
        CT(cudaMalloc(dr0, sizeof(int64_t) * (size_t)std::max<int64_t>(nt, 1)));
        CT(cudaMalloc(dln, sizeof(int32_t) * (size_t)std::max<int64_t>(nt, 1)));
        if (nt) {
            CT(cudaMemcpy(*dr0, r0, sizeof(int64_t) * nt, cudaMemcpyHostToDevice));
            CT(cudaMemcpy(*dln, ln, sizeof(int32_t) * nt, cudaMemcpyHostToDevice));
        }
        return ARR_OK;
    };
    int64_t covered = 0;
    for (int64_t t = 0; t < d->n_int_tiles; ++t) {
        if (d->int_len[t] < 1 || d->int_len[t] > 64 || d->int_row0[t] < 0 || d->int_row0[t] + d->int_len[t] > c->A.n)
            return cfail(c, ARR_EINVAL, "dist: bad interior tile");
        covered += d->int_len[t];
    }
    for (int64_t t = 0; t < d->n_bnd_tiles; ++t) {
        if (d->bnd_len[t] < 1 || d->bnd_len[t] > 64 || d->bnd_row0[t] < 0 || d->bnd_row0[t] + d->bnd_len[t] > c->A.n)
            return cfail(c, ARR_EINVAL, "dist: bad boundary tile");
        covered += d->bnd_len[t];
    }
    if (covered != c->A.n) return cfail(c, ARR_EINVAL, "dist: interior + boundary tiles must cover the owned rows");
    arr_status st;
    if ((st = up(d->int_row0, d->int_len, d->n_int_tiles, &P.int_row0, &P.int_len)) != ARR_OK) return st;
    if ((st = up(d->bnd_row0, d->bnd_len, d->n_bnd_tiles, &P.bnd_row0, &P.bnd_len)) != ARR_OK) return st;
    P.n_int_tiles = d->n_int_tiles;
    P.n_bnd_tiles = d->n_bnd_tiles;
    CT(cudaStreamCreateWithFlags(&P.comm_stream, cudaStreamNonBlocking));
    CT(cudaEventCreateWithFlags(&P.ev_ready, cudaEventDisableTiming));
    CT(cudaEventCreateWithFlags(&P.ev_done, cudaEventDisableTiming));
    if (m->kind == 1) {
        // staging for the in-process allreduce: the largest reduction is H (m x m)
        const int64_t mm = (int64_t)(c->p + 1) * c->w;
        c->stage_elems = (size_t)std::max<int64_t>(mm * mm, 2 * ARR_MAX_W + 64);
        CT(cudaMalloc(&c->stage, sizeof(double) * c->stage_elems));
        LocalSlot &me = m->group->slot[m->rank];
        me.ctx = c;
        if (!me.ready) CT(cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming));
        if (!me.done) CT(cudaEventCreateWithFlags(&me.done, cudaEventDisableTiming));
    }
    return ARR_OK;
}

void comm_free_plan(arr_ctx *c) {
    DistPlan &P = c->plan;
    void *ptrs[] = {P.send_rows_dev, P.sendbuf, P.recvbuf, P.int_row0, P.int_len, P.bnd_row0, P.bnd_len, c->stage};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (P.ev_ready) cudaEventDestroy(P.ev_ready);
    if (P.ev_done) cudaEventDestroy(P.ev_done);
    if (P.comm_stream) cudaStreamDestroy(P.comm_stream);
    if (c->comm && c->comm->kind == 1 && c->comm->group->slot[c->comm->rank].ctx == c)
        c->comm->group->slot[c->comm->rank].ctx = nullptr;
}

// ====================================================================== C-ABI
extern "C" {

arr_status comm_get_nccl_id(unsigned char *id_out) {
    if (!id_out) return ARR_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return ARR_ENCCL;
    memcpy(id_out, id.internal, NCCL_UNIQUE_ID_BYTES);
    return ARR_OK;
}

arr_status comm_init_nccl(arr_comm **out, const unsigned char *id, int32_t rank, int32_t size) {
    if (!out || !id || size < 1 || rank < 0 || rank >= size) return ARR_EINVAL;
    *out = nullptr;
    arr_comm *m = new (std::nothrow) arr_comm();
    if (!m) return ARR_ENOMEM;
    m->rank = rank;
    m->size = size;
    m->kind = 0;
    ncclUniqueId uid;
    memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
    if (ncclCommInitRank(&m->nccl, size, uid, rank) != ncclSuccess) {
        delete m;
        return ARR_ENCCL;
    }
    *out = m;
    return ARR_OK;
}

arr_status comm_init_local_group(arr_comm **out, int32_t size) {
    if (!out || size < 1 || size > kMaxRanks) return ARR_EINVAL;
    LocalGroup *g = new (std::nothrow) LocalGroup();
    if (!g) return ARR_ENOMEM;
    g->size = size;
    g->refs = size;
    g->slot.resize(size);
    for (int r = 0; r < size; ++r) {
        arr_comm *m = new (std::nothrow) arr_comm();
        if (!m) return ARR_ENOMEM;
        m->rank = r;
        m->size = size;
        m->kind = 1;
        m->group = g;
        out[r] = m;
    }
    return ARR_OK;
}

arr_status comm_destroy(arr_comm *m) {
    if (!m) return ARR_EINVAL;
    if (m->kind == 0) {
        if (m->nccl) ncclCommDestroy(m->nccl);
    } else {
        LocalGroup *g = m->group;
        bool last = false;
        {
            std::lock_guard<std::mutex> lk(g->m);
            last = (--g->refs == 0);
        }
        if (last) {
            for (auto &s : g->slot) {
                if (s.ready) cudaEventDestroy(s.ready);
                if (s.done) cudaEventDestroy(s.done);
            }
            delete g;
        }
    }
    delete m;
    return ARR_OK;
}

arr_status comm_rank_size(const arr_comm *m, int32_t *rank, int32_t *size) {
    if (!m || !rank || !size) return ARR_EINVAL;
    *rank = m->rank;
    *size = m->size;
    return ARR_OK;
}

}  // extern "C"
