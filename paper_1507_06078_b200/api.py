"""Thin Python binding over the C-ABI (include/arrabit.h), same names.

Blocks are torch fp64 CUDA tensors of shape (n, ncols) with stride (ld, 1)
(row-major, ld >= ncols).  The CSR arrays are torch CUDA tensors (int64 row_ptr,
int32 col_idx, fp64 val).  PyTorch only supplies device memory and streams;
every arithmetic step runs in libarrabit's kernels.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import arr_csr, arr_dist, arr_solve_info, arr_solve_opts


LOG_FIELDS = 12  # ARR_LOG_FIELDS (include/arrabit.h)
LOG_KEYS = ("outer", "s", "a", "b", "mu1", "maxres", "p", "d", "locked", "tol_t", "mu_k", "mu_w")


class ArrError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


@dataclass
class DeviceCSR:
    n: int
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    val: torch.Tensor

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())


def to_device_csr(A, device="cuda") -> DeviceCSR:
    """Copy a host CSR (fields n, row_ptr, col_idx, val as numpy) to the device."""
    return DeviceCSR(int(A.n),
                     torch.from_numpy(np.ascontiguousarray(A.row_ptr, dtype=np.int64)).to(device),
                     torch.from_numpy(np.ascontiguousarray(A.col_idx, dtype=np.int32)).to(device),
                     torch.from_numpy(np.ascontiguousarray(A.val, dtype=np.float64)).to(device))


def _blk(X: torch.Tensor, name: str):
    if X.dtype != torch.float64 or not X.is_cuda or X.dim() != 2 or X.stride(1) != 1:
        raise ValueError(f"{name}: need a row-major fp64 CUDA tensor (n, ncols) with stride (ld, 1)")
    return ctypes.c_void_p(X.data_ptr()), X.stride(0), X.shape[1]


def _stream_handle(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream), stream


class Comm:
    """An arr_comm: NCCL (one process per GPU) or one rank of an in-process group."""

    def __init__(self, handle: ctypes.c_void_p, owner=None):
        self.lib = _lib.load()
        self.h = handle
        self._owner = owner
        r, s = ctypes.c_int32(), ctypes.c_int32()
        self.lib.comm_rank_size(self.h, ctypes.byref(r), ctypes.byref(s))
        self.rank, self.size = r.value, s.value

    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = _lib.load()
        buf = ctypes.create_string_buffer(128)
        st = lib.comm_get_nccl_id(buf)
        if st != 0:
            raise ArrError(st, "comm_get_nccl_id failed")
        return buf.raw

    @classmethod
    def nccl(cls, uid: bytes, rank: int, size: int) -> "Comm":
        """Collective over the size ranks; the rank's device must be current."""
        lib = _lib.load()
        h = ctypes.c_void_p()
        st = lib.comm_init_nccl(ctypes.byref(h), uid, int(rank), int(size))
        if st != 0:
            raise ArrError(st, "comm_init_nccl failed")
        return cls(h)

    @classmethod
    def from_torch_distributed(cls) -> "Comm":
        """NCCL communicator over the default torch.distributed group (rank 0's
        unique id is broadcast with torch.distributed; the data path is NCCL
        inside libarrabit)."""
        import torch.distributed as dist
        obj = [cls.nccl_unique_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return cls.nccl(obj[0], dist.get_rank(), dist.get_world_size())

    @classmethod
    def local_group(cls, size: int) -> list["Comm"]:
        """size communicators of one in-process group (one host thread per rank)."""
        lib = _lib.load()
        arr = (ctypes.c_void_p * size)()
        st = lib.comm_init_local_group(arr, int(size))
        if st != 0:
            raise ArrError(st, "comm_init_local_group failed")
        return [cls(ctypes.c_void_p(arr[r])) for r in range(size)]

    def close(self):
        if getattr(self, "h", None):
            self.lib.comm_destroy(self.h)
            self.h = None


def _dist_struct(plan):
    """arr_dist from a partition.LocalPlan (host arrays; the library copies them)."""
    keep = []

    def p(a, dt):
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return ctypes.c_void_p(a.ctypes.data) if a.size else None

    d = arr_dist(plan.n_global, plan.row_begin, plan.n_ghost, len(plan.peer), p(plan.peer, np.int32),
                 p(plan.send_off, np.int64), p(plan.send_rows, np.int32), p(plan.recv_off, np.int64),
                 p(plan.int_row0, np.int64), p(plan.int_len, np.int32), len(plan.int_row0),
                 p(plan.bnd_row0, np.int64), p(plan.bnd_len, np.int32), len(plan.bnd_row0))
    return d, keep


class EigContext:
    """An arr_ctx (eig_init ... eig_destroy).  With ``comm`` and ``plan`` (a
    partition.LocalPlan whose local CSR is ``A``) it is one rank of a
    distributed context (eig_init_dist): every call is collective and every
    block has plan.n_rows_block rows."""

    def __init__(self, A: DeviceCSR, k: int, p: int, d: int, stream=None, w: int | None = None, comm=None,
                 plan=None):
        self.lib = _lib.load()
        self.A = A  # keep the borrowed arrays alive
        self.k, self.p, self.d = k, p, d
        self.w = k if w is None else w
        self.comm, self.plan = comm, plan
        self.handle_stream, self.stream = _stream_handle(stream)
        self._csr = arr_csr(A.n, A.nnz, A.row_ptr.data_ptr(), A.col_idx.data_ptr(), A.val.data_ptr())
        h = ctypes.c_void_p()
        if comm is not None:
            if plan is None:
                raise ValueError("a distributed context needs the rank's partition plan")
            ds, _keep = _dist_struct(plan)
            st = self.lib.eig_init_dist(ctypes.byref(h), ctypes.byref(self._csr), k, self.w, p, d, ctypes.byref(ds),
                                        comm.h, self.handle_stream)
        else:
            st = self.lib.eig_init_w(ctypes.byref(h), ctypes.byref(self._csr), k, self.w, p, d, self.handle_stream)
        if st != 0:
            raise ArrError(st, "eig_init failed")
        self.h = h

    # -- helpers
    def _check(self, st: int, what: str):
        if st != 0:
            msg = self.lib.eig_last_error(self.h)
            raise ArrError(st, f"{what}: {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.eig_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(self.lib.eig_launch_count(self.h))

    @property
    def workspace_bytes(self) -> int:
        return int(self.lib.eig_workspace_bytes(self.h))

    def eig_set_timing(self, on: bool = True):
        self._check(self.lib.eig_set_timing(self.h, 1 if on else 0), "eig_set_timing")

    def eig_phase_times(self):
        """(ms[6], counts[6]) for phases filter-degrees / arr_project / residuals /
        arr.basis / arr.H / arr.eig (see include/arrabit.h)."""
        ms = np.zeros(6)
        cnt = np.zeros(6, dtype=np.int64)
        self._check(self.lib.eig_phase_times(self.h, ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                             cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
                    "eig_phase_times")
        return ms, cnt

    def eig_kernel_times(self):
        """The FP64 DMMA kernels alone: (ms[2], flops[2], launches[2]) for the Gram (0) and
        GEMM (1) kernels since eig_set_timing(True), flops algorithmic (include/arrabit.h)."""
        ms = np.zeros(2)
        fl = np.zeros(2)
        cnt = np.zeros(2, dtype=np.int64)
        self._check(self.lib.eig_kernel_times(self.h, ms.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                              fl.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                              cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
                    "eig_kernel_times")
        return ms, fl, cnt

    # -- A0
    def eig_gershgorin_lower(self) -> float:
        a = ctypes.c_double()
        self._check(self.lib.eig_gershgorin_lower(self.h, ctypes.byref(a)), "eig_gershgorin_lower")
        return a.value

    def eig_set_interval(self, a: float, b: float):
        self._check(self.lib.eig_set_interval(self.h, float(a), float(b)), "eig_set_interval")

    def eig_set_schedule(self, tile_row0: np.ndarray | None, tile_len: np.ndarray | None = None):
        """Processing order of row tiles (see include/arrabit.h); None = natural order."""
        if tile_row0 is None:
            self._sched = None
            self._check(self.lib.eig_set_schedule(self.h, None, None, 0), "eig_set_schedule")
            return
        r0 = torch.from_numpy(np.ascontiguousarray(tile_row0, dtype=np.int64)).to(self.A.row_ptr.device)
        ln = torch.from_numpy(np.ascontiguousarray(tile_len, dtype=np.int32)).to(self.A.row_ptr.device)
        self._sched = (r0, ln)  # keep the borrowed arrays alive
        self._check(self.lib.eig_set_schedule(self.h, ctypes.c_void_p(r0.data_ptr()), ctypes.c_void_p(ln.data_ptr()),
                                              int(r0.numel())), "eig_set_schedule")

    def eig_set_stencil(self, nx: int, ny: int = 1, nz: int = 1):
        """Declare A a <= 27-point stencil on an nx x ny x nz grid (x fastest); (0, 0, 0)
        switches back to the CSR kernels (see include/arrabit.h)."""
        self._check(self.lib.eig_set_stencil(self.h, int(nx), int(ny), int(nz)), "eig_set_stencil")

    @property
    def last_spmm_kernel(self) -> str:
        """Name of the kernel the last fused SpMM of this context launched."""
        return self.lib.eig_last_spmm_kernel(self.h).decode()

    @property
    def stencil_points(self) -> int:
        """K of the active stencil path (0: CSR kernels)."""
        return int(self.lib.eig_stencil_active(self.h))

    @property
    def stencil_abytes(self) -> int:
        """Bytes of A per row the stencil path reads (8 K, 8 or 0; -1: no stencil)."""
        return int(self.lib.eig_stencil_abytes(self.h))

    def eig_set_degree(self, d: int):
        self._check(self.lib.eig_set_degree(self.h, int(d)), "eig_set_degree")
        self.d = d

    def eig_set_mode(self, which: str = "largest"):
        """'largest' (default) or 'smallest' k eigenpairs (see include/arrabit.h)."""
        self._check(self.lib.eig_set_mode(self.h, 1 if which == "smallest" else 0), "eig_set_mode")

    FILTERS = {"cheb": 0, "interp": 1}

    def eig_set_filter(self, kind: str = "cheb"):
        """'cheb': T_d of the mapped matrix (default); 'interp': the paper's psi_d
        (Chebyshev interpolant of max(0,t)^{10d}, see include/arrabit.h)."""
        self._check(self.lib.eig_set_filter(self.h, self.FILTERS[kind]), "eig_set_filter")

    # -- A1/A2
    def filter_step(self, X: torch.Tensor, normalize: bool | str = True, colnorm: torch.Tensor | None = None):
        """normalize: True (unit columns), False, or "lazy" (norms pending for the next
        filter_step on the same X, include/arrabit.h)."""
        px, ld, _ = _blk(X, "X")
        cn = ctypes.c_void_p(colnorm.data_ptr()) if colnorm is not None else None
        mode = 2 if normalize == "lazy" else (1 if normalize else 0)
        self._check(self.lib.filter_step(self.h, px, ld, mode, cn), "filter_step")

    # -- A3
    def spmm(self, X: torch.Tensor, Y: torch.Tensor, alpha: float = 1.0, shift: float = 0.0):
        px, ldx, nc = _blk(X, "X")
        py, ldy, nc2 = _blk(Y, "Y")
        if nc2 != nc:
            raise ValueError("spmm: column mismatch")
        self._check(self.lib.spmm(self.h, float(alpha), float(shift), px, ldx, py, ldy, nc), "spmm")

    # -- A4
    def gram(self, X: torch.Tensor, Y: torch.Tensor, G: torch.Tensor):
        px, ldx, m1 = _blk(X, "X")
        py, ldy, m2 = _blk(Y, "Y")
        pg, ldg, _ = _blk(G, "G")
        self._check(self.lib.gram(self.h, px, ldx, m1, py, ldy, m2, pg, ldg), "gram")

    def gemm(self, X: torch.Tensor, B: torch.Tensor, Out: torch.Tensor, alpha: float = 1.0, beta: float = 0.0,
             Cin: torch.Tensor | None = None):
        px, ldx, m1 = _blk(X, "X")
        pb, ldb, m2 = _blk(B, "B")
        po, ldo, _ = _blk(Out, "Out")
        if Cin is not None:
            pc, ldc, _ = _blk(Cin, "Cin")
        else:
            pc, ldc = None, 0
        self._check(self.lib.gemm(self.h, float(alpha), px, ldx, m1, pb, ldb, m2, float(beta), pc, ldc, po, ldo),
                    "gemm")

    def orthonormalize(self, X: torch.Tensor) -> int:
        px, ld, nc = _blk(X, "X")
        r = ctypes.c_int32()
        self._check(self.lib.orthonormalize(self.h, px, ld, nc, ctypes.byref(r)), "orthonormalize")
        return r.value

    def arr_project(self, X: torch.Tensor, Y: torch.Tensor | None = None, p: int | None = None):
        p = self.p if p is None else p
        px, ldx, _ = _blk(X, "X")
        if Y is not None:
            py, ldy, _ = _blk(Y, "Y")
        else:
            py, ldy = None, 0
        ritz = np.empty((p + 1) * self.w)
        r = ctypes.c_int32()
        self._check(self.lib.arr_project_p(self.h, p, px, ldx, py, ldy,
                                           ritz.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(r)),
                    "arr_project")
        return ritz, r.value

    # -- A6
    def residuals(self, Y: torch.Tensor, mu) -> np.ndarray:
        py, ldy, nc = _blk(Y, "Y")
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        if len(mu) != nc:
            raise ValueError("residuals: len(mu) != ncols")
        res = np.empty(nc)
        self._check(self.lib.residuals(self.h, py, ldy, mu.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nc,
                                       res.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), "residuals")
        return res

    # -- driver
    def eig_solve(self, X: torch.Tensor, tol: float = 1e-10, maxit: int = 300, s_max: int = 5, exits: int = 0,
                  inner: str = "range", adapt: int = 0, inner_solver: str = "mpm", range_digits: float = 0.0):
        """exits: the paper's extra stop rules as a bit mask: 1 = (ii), 2 = (iii).
        inner: 'range' (dynamic-range rule, R6) or 'rcond' (the paper's).
        range_digits: D of the dynamic-range rule (0 = the library default, 12).
        adapt: the paper's adaptive p (bit 1), degree (bit 2), continuation + deflation (bit 4).
        inner_solver: 'mpm' (default) or 'gn' (Gauss-Newton, Alg. Arrabit2)."""
        px, ld, _ = _blk(X, "X")
        opts = arr_solve_opts(tol, maxit, s_max, exits, 1 if inner == "rcond" else 0, adapt,
                              1 if inner_solver == "gn" else 0)
        log = np.zeros((maxit, LOG_FIELDS))
        opts.log = ctypes.c_void_p(log.ctypes.data)
        opts.log_cap = maxit
        opts.range_digits = range_digits
        ev = np.empty(self.k)
        res = np.empty(self.k)
        info = arr_solve_info()
        self._check(self.lib.eig_solve(self.h, px, ld, ctypes.byref(opts),
                                       ev.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                       res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(info)),
                    "eig_solve")
        n = min(int(info.outer), maxit)
        self.last_log = [dict(zip(LOG_KEYS, row)) for row in log[:n]]
        return ev, res, info


class ColSplitContext(EigContext):
    """A column-partitioned context (eig_init_colsplit): blocks are this rank's column
    slice (n x w_r, all rows); A_full is the whole matrix on every rank, A_rows and
    ``plan`` (partition.ColSplitPlan) the row block of the internal ARR context."""

    def __init__(self, A_full: DeviceCSR, A_rows: DeviceCSR, plan, k: int, p: int, d: int, w: int, comm,
                 stream=None):
        self.lib = _lib.load()
        self.A, self.A_rows = A_full, A_rows
        self.k, self.p, self.d, self.w = k, p, d, w
        self.comm, self.plan = comm, plan
        self.handle_stream, self.stream = _stream_handle(stream)
        self._csr = arr_csr(A_full.n, A_full.nnz, A_full.row_ptr.data_ptr(), A_full.col_idx.data_ptr(),
                            A_full.val.data_ptr())
        self._csr_rows = arr_csr(A_rows.n, A_rows.nnz, A_rows.row_ptr.data_ptr(), A_rows.col_idx.data_ptr(),
                                 A_rows.val.data_ptr())
        ds, _keep = _dist_struct(plan.rows)
        self._rb = np.ascontiguousarray(plan.row_begins, dtype=np.int64)
        self._cb = np.ascontiguousarray(plan.col_begins, dtype=np.int64)
        h = ctypes.c_void_p()
        st = self.lib.eig_init_colsplit(ctypes.byref(h), ctypes.byref(self._csr), k, w, p, d,
                                        ctypes.byref(self._csr_rows), ctypes.byref(ds),
                                        ctypes.c_void_p(self._rb.ctypes.data), ctypes.c_void_p(self._cb.ctypes.data),
                                        comm.h, self.handle_stream)
        if st != 0:
            raise ArrError(st, "eig_init_colsplit failed")
        self.h = h

    def residuals(self, Y: torch.Tensor, mu) -> np.ndarray:
        """Residuals of the first len(mu) pairs; Y is this rank's column slice of the block."""
        py, ldy, _ = _blk(Y, "Y")
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        res = np.empty(len(mu))
        self._check(self.lib.residuals(self.h, py, ldy, mu.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(mu),
                                       res.ctypes.data_as(ctypes.POINTER(ctypes.c_double))), "residuals")
        return res

    @property
    def w_local(self) -> int:
        c0, c1 = self.plan.col_range
        return c1 - c0


def eig_init_colsplit(A_full: DeviceCSR, A_rows: DeviceCSR, plan, k: int, p: int, d: int, w: int, comm,
                      stream=None) -> ColSplitContext:
    return ColSplitContext(A_full, A_rows, plan, k, p, d, w, comm, stream)


def eig_init(A: DeviceCSR, k: int, p: int, d: int, stream=None, w: int | None = None, comm=None,
             plan=None) -> EigContext:
    """eig_init (w = k) / eig_init_w (w >= k guard columns) / eig_init_dist (comm + plan)."""
    return EigContext(A, k, p, d, stream, w, comm, plan)


def eig_solve_host(n, row_ptr, col_idx, val, k, p, d, X0, tol=1e-10, maxit=300, s_max=5, evec=None,
                   stream=None, grid=None):
    """Public host-buffer entry (eig_solve_host): host arrays in, host results out.
    X0 is n x w (w >= k; w - k guard columns).  Arguments may be numpy arrays or
    (pinned) CPU torch tensors.  grid = (nx, ny, nz) declares A a stencil operator
    (eig_set_stencil on the internal context)."""
    lib = _lib.load()
    w = int(X0.shape[1])

    def ptr(a):
        if isinstance(a, torch.Tensor):
            assert not a.is_cuda and a.is_contiguous()
            return ctypes.c_void_p(a.data_ptr())
        assert a.flags.c_contiguous
        return ctypes.c_void_p(a.ctypes.data)

    nnz = int(col_idx.shape[0])
    ev = np.empty(k)
    res = np.empty(k)
    info = arr_solve_info()
    opts = arr_solve_opts(tol, maxit, s_max, 0, 0, 0, 0)
    if grid is not None:
        opts.grid[0], opts.grid[1], opts.grid[2] = (int(x) for x in grid)
    hs, _ = _stream_handle(stream)
    st = lib.eig_solve_host(int(n), nnz, ptr(row_ptr), ptr(col_idx), ptr(val), k, w, p, d, ptr(X0),
                            ctypes.byref(opts), ev.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            res.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            ptr(evec) if evec is not None else None, ctypes.byref(info), hs)
    if st != 0:
        raise ArrError(st, "eig_solve_host failed")
    return ev, res, info
