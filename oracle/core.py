"""ORACLE — test infrastructure only (see oracle/__init__.py).

Plain fp64 CPU implementation of the ARRABIT-MPM hot path, arXiv 1507.06078
(P = /root/reference/PAPER.md line numbers; readings in DESIGN.md §4).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import sys
from dataclasses import dataclass, field

import numpy as np

from . import dense

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)


def build_lib(force: bool = False) -> str:
    """Compile csr_oracle.c -> liboracle.so (plain gcc, -O2, OpenMP, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


def load_lib():
    global _lib
    if _lib is None:
        build_lib()
        lib = ctypes.CDLL(_LIB)
        lib.orc_spmm.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i32p, _f64p,
                                 _f64p, ctypes.c_int64, _f64p, ctypes.c_int64]
        lib.orc_spmm.restype = None
        lib.orc_cheb_filter.argtypes = [ctypes.c_int64, ctypes.c_int64, _i64p, _i32p, _f64p,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int32,
                                        _f64p, ctypes.c_int64, _f64p, ctypes.c_int64]
        lib.orc_cheb_filter.restype = ctypes.c_int
        lib.orc_col_norms.argtypes = [ctypes.c_int64, ctypes.c_int64, _f64p, ctypes.c_int64, _f64p]
        lib.orc_col_norms.restype = None
        _lib = lib
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _csr_args(A):
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int32)
    va = np.ascontiguousarray(A.val, dtype=np.float64)
    return rp, ci, va


# --------------------------------------------------------------------------- sparse
def spmm(A, X: np.ndarray) -> np.ndarray:
    """Y = A X (plain CSR row loop in C).  P:1527-1528: A enters only through AX."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    if X.ndim == 1:
        return spmm(A, X[:, None])[:, 0]
    n, w = X.shape
    if n != A.n:
        raise ValueError("dimension mismatch")
    Y = np.empty_like(X)
    rp, ci, va = _csr_args(A)
    load_lib().orc_spmm(n, w, _p(rp, _i64p), _p(ci, _i32p), _p(va, _f64p),
                        _p(X, _f64p), w, _p(Y, _f64p), w)
    return Y


def cheb_filter(A, a: float, b: float, d: int, X: np.ndarray) -> np.ndarray:
    """Y = T_d((A - cI)/e) X, c=(a+b)/2, e=(b-a)/2 (Eq. cheby-poly P:377-383 on the
    affine map of Eq. rhod; reading DESIGN.md §4 R1/R2)."""
    if not a < b:
        raise ValueError("need a < b")
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, w = X.shape
    Y = np.empty_like(X)
    rp, ci, va = _csr_args(A)
    rc = load_lib().orc_cheb_filter(n, w, _p(rp, _i64p), _p(ci, _i32p), _p(va, _f64p),
                                    float(a), float(b), int(d), _p(X, _f64p), w, _p(Y, _f64p), w)
    if rc != 0:
        raise RuntimeError(f"orc_cheb_filter failed ({rc})")
    return Y


def col_norms(X: np.ndarray) -> np.ndarray:
    X = np.ascontiguousarray(X, dtype=np.float64)
    n, w = X.shape
    out = np.empty(w)
    load_lib().orc_col_norms(n, w, _p(X, _f64p), w, _p(out, _f64p))
    return out


def mpm_sweep(A, a: float, b: float, d: int, X: np.ndarray) -> np.ndarray:
    """One multi-power sweep: x_i <- rho(A) x_i, x_i <- x_i/||x_i||_2 for every
    column, no orthogonalisation (Alg. Arrabit2)."""
    Y = cheb_filter(A, a, b, d, X)
    nrm = col_norms(Y)
    if np.any(nrm == 0) or not np.all(np.isfinite(nrm)):
        raise FloatingPointError("zero or non-finite column after filtering")
    return Y / nrm


def gershgorin_lower(A) -> float:
    """a = min_i (A_ii - sum_{j != i} |A_ij|): a lower bound of lambda_n, used
    in place of the paper's eigs call (reading DESIGN.md §4 R3)."""
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    diag = np.zeros(A.n)
    off = np.zeros(A.n)
    isd = A.col_idx == rows
    np.add.at(diag, rows[isd], A.val[isd])
    np.add.at(off, rows[~isd], np.abs(A.val[~isd]))
    return float(np.min(diag - off))


def chebyshev_T(d: int, t):
    """rho_d(t) by the three-term recursion rho_{d+1} = 2 t rho_d - rho_{d-1},
    rho_0 = 1, rho_1 = t (Eq. cheby-poly)."""
    t = np.asarray(t, dtype=np.float64)
    r0 = np.ones_like(t)
    if d == 0:
        return r0
    r1 = t.copy()
    for _ in range(1, d):
        r0, r1 = r1, 2.0 * t * r1 - r0
    return r1


def interp_coeffs(d: int) -> np.ndarray:
    """Chebyshev coefficients a_0..a_d of psi_d(t) = sum_k a_k T_k(t), the degree-d
    Chebyshev interpolant of f_d(t) = max(0, t)^{10 d} (Eq. def:fN,
    P:1198-1202) at the points of the second kind t_j = -cos(j pi / d), j = 0..d
    (P:1186-1189).  The interpolant is unique, so it is written as the solution of
    the square collocation system sum_k a_k T_k(t_j) = f_d(t_j) (one library solve).
    Reading (R18): psi_d is kept in the Chebyshev basis; the paper's
    monomial coefficients Gamma_d (Eq. chebfun-f) reach 1e5 (d = 20) and 3e8 (d = 30)
    with alternating signs, so two fp64 computations of them differ by 1e-11 to 1e-7
    relative and Alg. poly's Horner output by up to 1e-4 — not a reproducible target.
    The square system is solved by the oracle's own Gaussian elimination (dense.solve_gepp)."""
    if d < 1:
        raise ValueError("d >= 1")
    t = -np.cos(np.arange(d + 1) * np.pi / d)
    f = np.maximum(0.0, t) ** (10 * d)
    return dense.solve_gepp(chebyshev_basis(d, t), f)


def chebyshev_basis(d: int, t) -> np.ndarray:
    """[T_0(t), .., T_d(t)] as columns (three-term recursion, Eq. cheby-poly)."""
    t = np.asarray(t, dtype=np.float64)
    B = np.empty((t.size, d + 1))
    for k in range(d + 1):
        B[:, k] = chebyshev_T(k, t)
    return B


def psi(coef: np.ndarray, t):
    """psi_d(t) = sum_k a_k T_k(t) (plain sum over the basis)."""
    t = np.asarray(t, dtype=np.float64)
    return chebyshev_basis(len(coef) - 1, t.ravel()).dot(coef).reshape(t.shape)


def poly_filter(A, a: float, b: float, coef: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Y = rho_d(A) X with rho_d(t) = psi_d(c_0 + c_1 t), c_0 = (a+b)/(a-b),
    c_1 = 2/(b-a) (Eq. rhod; the map of Alg. poly), evaluated by
    Clenshaw's recurrence in the Chebyshev basis with S = c_1 A + c_0 I:
        b_{d+1} = b_{d+2} = 0,  b_k = a_k X + 2 S b_{k+1} - b_{k+2}  (k = d .. 1),
        Y = a_0 X + S b_1 - b_2."""
    if not a < b:
        raise ValueError("need a < b")
    X = np.ascontiguousarray(X, dtype=np.float64)
    c0 = (a + b) / (a - b)
    c1 = 2.0 / (b - a)
    d = len(coef) - 1

    def S(V):
        return c1 * spmm(A, V) + c0 * V

    b2 = np.zeros_like(X)
    b1 = np.zeros_like(X)
    for k in range(d, 0, -1):
        b1, b2 = coef[k] * X + 2.0 * S(b1) - b2, b1
    return coef[0] * X + S(b1) - b2


def poly_sweep(A, a: float, b: float, coef: np.ndarray, X: np.ndarray) -> np.ndarray:
    """One multi-power sweep with the paper's filter: rho_d(A) then column normalisation
    (Alg. Arrabit2)."""
    Y = poly_filter(A, a, b, coef, X)
    nrm = col_norms(Y)
    if np.any(nrm == 0) or not np.all(np.isfinite(nrm)):
        raise FloatingPointError("zero or non-finite column after filtering")
    return Y / nrm


def gn_step(A, a: float, b: float, d: int, X: np.ndarray, coef=None) -> np.ndarray:
    """One Gauss-Newton inner step of Alg. Arrabit2 (Alg. GN) with
    the accelerator rho_d in place of A: Y = X (X^T X)^{-1}; Z = rho_d(A) Y;
    X = Z - X (Y^T Z - I) / 2.  rho_d = T_d of the mapped matrix (coef None) or psi_d."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    R = dense.cholesky_upper(dense.gram(X, X))          # X^T X = R^T R
    Rinv = dense.solve_upper_right(np.eye(R.shape[0]), R)
    Y = dense.gemm(X, Rinv @ Rinv.T)                     # X (X^T X)^{-1}
    Z = cheb_filter(A, a, b, d, Y) if coef is None else poly_filter(A, a, b, coef, Y)
    return Z - X @ (Y.T @ Z - np.eye(X.shape[1])) / 2.0


# --------------------------------------------------------------------------- dense
def orthonormalize(Z: np.ndarray):
    """U in orth(Z) (Alg. RR step 1): equilibrate columns (span unchanged),
    Householder QR with column pivoting (the oracle's own, dense.qr_pivoted), keep
    r = #{i : |R_ii| > n*eps*|R_11|} columns (reading DESIGN.md R8)."""
    Z = np.asarray(Z, dtype=np.float64)
    n, m = Z.shape
    nrm = np.sqrt(np.einsum("ij,ij->j", Z, Z))
    keep = nrm > 0
    Zs = Z[:, keep] / nrm[keep]
    if Zs.shape[1] == 0:
        return np.zeros((n, 0)), 0
    Q, R, _ = dense.qr_pivoted(Zs)
    dR = np.abs(np.diag(R))
    r = int(np.sum(dR > n * np.finfo(float).eps * dR[0]))
    return Q[:, :r], r


# Eigen-decomposition of the small projected matrix H (Alg. RR step 3): the
# oracle's own cyclic Jacobi (dense.jacobi_eigh) everywhere, except where a caller sets
# EIGH = "lapack" (numpy.linalg.eigh as a library step): only scripts/oracle_golden.py does,
# for the m = 1650 problems of the full cfg3 solve, where the numpy Jacobi takes ~25 minutes
# per ARR.  The two are cross-checked in tests/test_oracle_own_dense.py.
EIGH = "jacobi"


def _ritz(A, U: np.ndarray, H: np.ndarray | None = None):
    """Alg. RR steps 2-4 on an orthonormal U: H = U^T A U (symmetrised),
    H = V Sigma V^T by cyclic Jacobi (dense.jacobi_eigh), Ritz values descending,
    Y = U V."""
    if H is None:
        H = U.T @ spmm(A, U) if U.shape[1] > 0 else np.zeros((0, 0))
    H = 0.5 * (H + H.T)
    mu, V = dense.jacobi_eigh(H) if EIGH == "jacobi" else np.linalg.eigh(H)
    order = np.argsort(-mu, kind="stable")
    return mu[order], V[:, order]


def rayleigh_ritz(A, Z: np.ndarray):
    """(Y, Sigma) = RR(A, Z), Alg. RR: U = orth(Z); H = U^T A U;
    H = V^T Sigma V; Y = U V.  Ritz values sorted descending."""
    U, r = orthonormalize(Z)
    mu, V = _ritz(A, U)
    return mu, U @ V, r


def _top_up(Y: np.ndarray, keep: int, rng_seed: int):
    """Fill a rank-deficient Ritz block to `keep` columns with seeded Gaussian columns
    orthonormalised against it (reading DESIGN.md R7)."""
    n, r = Y.shape
    extra = np.random.default_rng(rng_seed).standard_normal((n, keep - r))
    for _ in range(2):
        extra -= Y @ (Y.T @ extra)
    Qe, _ = dense.qr_blocked(extra)
    return np.hstack([Y, Qe])


def arr(A, X: np.ndarray, p: int, keep: int | None = None, rng_seed: int = 12345, method: str = "qr",
        Qc: np.ndarray | None = None):
    """(Y, Sigma) = ARR(A, X, p), Alg. ARR, returns (mu_all_descending,
    Y_keep, rank).

    method "qr" (paper-literal): Z = [X, AX, ..., A^p X] with plain A (Eq. S:ARR,
      P:515-523), RR(A, Z) with the pivoted-QR orth.
    method "cgs2" (the orthonormalise-then-augment reading R8, the GPU's span):
      U_0 = orth(X), U_j = orth((I - Q Q^T) A U_{j-1}) with block classical Gram-Schmidt
      applied twice (row-panel Gram / GEMM loops, dense.gram / dense.gemm) and orth = the
      oracle's blocked Householder QR; if max |Q^T U_j| > 1e-12 (a nearly invariant block)
      U_j is projected out of Q twice more and re-orthonormalised; H = Q^T A Q one
      block column at a time (A Q never stored); RR steps 3-4.
    Qc (deflation): the ARR is performed in the orthogonal complement of
      R(Qc): every block of Z (qr) / every augmentation block (cgs2) has Qc projected out
      twice.
    If the rank r < keep the block is topped up with seeded Gaussian columns
    orthonormalised against Y (reading DESIGN.md R7)."""
    n, w = X.shape
    keep = w if keep is None else keep
    if (p + 1) * w >= n:
        raise ValueError("(p+1)k must be < n (Alg. ARR input, P:536)")

    def defl(B):
        if Qc is not None and Qc.shape[1] > 0:
            for _ in range(2):
                B = B - dense.gemm(Qc, dense.gram(Qc, B))
        return B

    if method == "qr":
        blocks = [np.asarray(X, dtype=np.float64)]
        for _ in range(p):
            blocks.append(spmm(A, blocks[-1]))
        Z = defl(np.hstack(blocks))
        mu, Y, r = rayleigh_ritz(A, Z)
    elif method == "cgs2":
        U, _ = dense.qr_blocked(np.asarray(X, dtype=np.float64))
        Q = U
        for j in range(1, p + 1):
            W = defl(spmm(A, Q[:, (j - 1) * w:j * w]))
            for _ in range(2):
                W = W - dense.gemm(Q, dense.gram(Q, W))
            Uj, _ = dense.qr_blocked(W)
            if np.max(np.abs(dense.gram(Q, Uj))) > 1e-12:
                for _ in range(2):
                    Uj = Uj - dense.gemm(Q, dense.gram(Q, Uj))
                Uj, _ = dense.qr_blocked(Uj)
            Q = np.hstack([Q, Uj])
        m = Q.shape[1]
        H = np.empty((m, m))
        for j in range(p + 1):
            H[:, j * w:(j + 1) * w] = dense.gram(Q, spmm(A, Q[:, j * w:(j + 1) * w]))
        mu, V = _ritz(A, Q, H)
        Y = dense.gemm(Q, V[:, :keep])
        r = m
    else:
        raise ValueError(method)
    if r >= keep:
        return mu, Y[:, :keep], r
    return mu, _top_up(Y, keep, rng_seed), r


def residuals(A, Y: np.ndarray, mu: np.ndarray) -> np.ndarray:
    """res_i = ||A y_i - mu_i y_i||_2 / max(1, |mu_i|)  (Eq. resi)."""
    AY = spmm(A, Y)
    R = AY - Y * mu[None, :]
    return col_norms(R) / np.maximum(1.0, np.abs(mu))


RANGE_DIGITS = 12.0  # D of the dynamic-range rule (R6)


def sweeps_rule(mu1: float, a: float, b: float, d: int, s_max: int, gamma=None,
                digits: float = RANGE_DIGITS) -> int:
    """Sweeps between ARR steps (DESIGN.md §4 R6, the dynamic-range rule that
    replaces the paper's rcond inner stop P:1355-1388): amp = |T_d((mu_1-c)/e)|
    (|psi_d((mu_1-c)/e)| with the interpolant filter),
    s = s_max if amp <= 1 else clamp(floor(D/log10(amp)), 1, s_max), D = digits."""
    c = 0.5 * (a + b)
    e = 0.5 * (b - a)
    t = (mu1 - c) / e
    amp = abs(float(chebyshev_T(d, t) if gamma is None else psi(gamma, np.array([t]))[0]))
    if not amp > 1.0:
        return s_max
    if not math.isfinite(amp):
        return 1
    return int(min(max(math.floor(digits / math.log10(amp)), 1), s_max))


@dataclass
class SolveResult:
    mu: np.ndarray
    Y: np.ndarray
    res: np.ndarray
    converged: bool
    outer: int
    sweeps: int
    log: list = field(default_factory=list)
    exit_rule: int = 0
    p_final: int = 0
    d_final: int = 0
    locked: int = 0


def rcond_gram(X: np.ndarray) -> float:
    """rc = lambda_min(X^T X) / lambda_max(X^T X), the reciprocal 2-norm condition of
    the Gram (the paper's rcond(X^T X), takes LAPACK's 1-norm estimate;
    reading DESIGN.md R6), eigenvalues by the oracle's Jacobi."""
    lam, _ = dense.jacobi_eigh(dense.gram(X, X))
    return max(lam[0], 0.0) / lam[-1] if lam[-1] > 0 else 0.0


def _degree_rule(d_max: int, a: float, b: float, mu_k: float, mu_w: float, gamma_of=None) -> int:
    """Eqs. hat-d / degree: the smallest d >= 3 with
    |rho_d(mu*_{k+q})| < 0.9 |rho_d(mu*_k)|, capped at d_max (rho_d = T_d on the
    interval map, or psi_d with the interpolant filter)."""
    c = 0.5 * (a + b)
    e = 0.5 * (b - a)
    for dd in range(3, d_max + 1):
        if gamma_of is None:
            rk = float(chebyshev_T(dd, (mu_k - c) / e))
            rw = float(chebyshev_T(dd, (mu_w - c) / e))
        else:
            g = gamma_of(dd)
            rk = float(psi(g, np.array([(mu_k - c) / e]))[0])
            rw = float(psi(g, np.array([(mu_w - c) / e]))[0])
        if abs(rw) < 0.9 * abs(rk):
            return dd
    return d_max


def solve(A, k: int, d: int, p: int, X0: np.ndarray, tol: float = 1e-10, maxit: int = 300,
          s_max: int = 5, w: int | None = None, max_outer: int | None = None, filter: str = "cheb",
          inner_solver: str = "mpm", arr_method: str = "qr", inner: str = "range", exits: int = 0,
          adapt: int = 0, range_digits: float = RANGE_DIGITS) -> SolveResult:
    """ARRABIT-MPM (Alg. Arrabit2).  Defaults = the fixed-parameter solve
    (adaptive lines disabled; R3/R6/R10):

        a := Gershgorin lower bound;  U0 := orth(X0); mu := eig(U0^T A U0); b := mu_w
        loop: s := sweeps_rule(mu_1);  s x { X := T_d((A-cI)/e) X; normalise }
              (mu, Y) := ARR(A, X, p)
              res_i, i <= k  (Eq. resi)  ;  stop if max res <= tol              (Eq. out-stop)
              b := mu_{w+1} (monotone once maxres grew);  X := Y[:, :w]   (R3)

    Options (the paper's rules, Section 6):
      inner="rcond": every maxit_2 = 5 sweeps (at most maxit_1 = 10 times) rc = rcond(X^T X);
        stop at rc <= tol or rc / rc_prev > 0.99 (Eq. inn-stop).
      exits bit 1: (ii) max res not reduced over three consecutive outer iterations;
            bit 2: (iii) max res < (1 + 9h/k) tol, h = #{res_i < 0.1 tol}.
      adapt bit 1: p from 1 up to p by Eq. block with the ratio taken on the
              shifted Ritz values (mu - a) (the inner solvers run on A - aI, P:1355-1357;
              DESIGN.md R20);
            bit 2: d from 3, re-chosen after every ARR by Eqs. hat-d / degree
              with d as d_max;
            bit 4: continuation + deflation (solve_deflate, R19).
      arr_method: "qr" (paper-literal) or "cgs2" (orthonormalise-then-augment, R8).
      range_digits: D of the dynamic-range rule (R6)."""
    if adapt & 4:
        if (adapt & 3) or inner != "range" or exits or inner_solver != "mpm":
            raise ValueError("continuation + deflation runs fixed p / d MPM sweeps only")
        return solve_deflate(A, k, d, p, X0, tol=tol, maxit=maxit, s_max=s_max, w=w, filter=filter,
                             arr_method=arr_method, max_outer=max_outer, range_digits=range_digits)
    n = A.n
    w = X0.shape[1] if w is None else w  # w - k guard vectors
    d_max, p_max = d, p
    gamma_of = None if filter == "cheb" else interp_coeffs  # "interp": the paper's psi_d (R18)
    p_cur = min(1, p_max) if adapt & 1 else p_max
    d_cur = 3 if (adapt & 2) and d_max > 3 else d_max
    X = np.array(X0[:, :w], dtype=np.float64, copy=True)
    a = gershgorin_lower(A)
    mu0, _, _ = arr(A, X, 0, method=arr_method)  # RR(A, X0) = ARR with p = 0
    b = float(mu0[w - 1])
    if not a < b:
        a = b - 1e-8 * (abs(b) + 1.0)
    mu1 = float(mu0[0])
    log = []
    sweeps = 0
    limit = maxit if max_outer is None else min(maxit, max_outer)
    mu = mu0
    Y = X
    res = np.full(k, np.inf)
    mono, prev_maxres = False, None
    hist = []
    best_res, best_muk, best_muw, maxresp = np.inf, 0.0, 0.0, np.inf
    exit_rule = 0

    def sweep(X):
        gamma = None if gamma_of is None else gamma_of(d_cur)
        if inner_solver == "gn":  # Alg. Arrabit2's GN branch
            return gn_step(A, a, b, d_cur, X, gamma)
        return mpm_sweep(A, a, b, d_cur, X) if gamma is None else poly_sweep(A, a, b, gamma, X)

    for outer in range(1, limit + 1):
        if inner == "rcond":
            s, rcp = 0, -1.0
            for _ in range(10):
                for _ in range(5):
                    X = sweep(X)
                s += 5
                rc = rcond_gram(X)
                if rc <= tol or (rcp > 0.0 and rc / rcp > 0.99):
                    break
                rcp = rc
        else:
            s = sweeps_rule(mu1, a, b, d_cur, s_max, None if gamma_of is None else gamma_of(d_cur), range_digits)
            for _ in range(s):
                X = sweep(X)
        sweeps += s
        mu, Y, r = arr(A, X, p_cur, keep=w, method=arr_method)
        res = residuals(A, Y[:, :k], mu[:k])
        maxres = float(np.max(res))
        log.append(dict(outer=outer, s=s, a=a, b=b, mu1=float(mu[0]), rank=r, maxres=maxres, p=p_cur, d=d_cur))
        if os.environ.get("ORACLE_VERBOSE"):  # progress of the hour-long golden solves (no arithmetic)
            print(log[-1], file=sys.stderr, flush=True)
        if maxres <= tol:
            return SolveResult(mu[:k].copy(), Y[:, :k].copy(), res, True, outer, sweeps, log, 1, p_cur, d_cur)
        if exits & 1:
            hist.append(maxres)
            h = len(hist)
            if h >= 4 and not (hist[h - 1] < hist[h - 4] or hist[h - 2] < hist[h - 4] or hist[h - 3] < hist[h - 4]):
                exit_rule = 2
                break
        if exits & 2:
            hsmall = int(np.sum(res < 0.1 * tol))
            if maxres < (1.0 + 9.0 * hsmall / k) * tol:
                exit_rule = 3
                break
        # b := mu_{w+1}, an under-estimate of lambda_{k+q} (mu_{w+1} <= lambda_{w+1} by
        # interlacing); once the max residual has grown tenfold between two
        # outer iterations (b fell and amplified the guard range), b only increases (R3)
        mono = mono or (prev_maxres is not None and maxres > 10.0 * prev_maxres)
        prev_maxres = maxres
        bn = float(mu[min(w, r - 1)])
        b = max(b, bn) if mono else bn
        if not a < b:
            a = b - 1e-8 * (abs(b) + 1.0)
        mu1 = float(mu[0])
        X = Y[:, :w]
        if maxres < best_res:
            best_res, best_muk, best_muw = maxres, float(mu[k - 1]), float(mu[w - 1])
        if (adapt & 1) and p_cur < p_max:  # Eq. block
            if (mu[w - 1] - a) / (mu[k - 1] - a) > 0.95 and maxres / maxresp > 0.1:
                p_cur += 1
        maxresp = maxres
        if (adapt & 2) and d_max > 3:  # Eqs. hat-d / degree
            d_cur = _degree_rule(d_max, a, b, best_muk, best_muw, gamma_of)
    return SolveResult(mu[:k].copy(), Y[:, :k].copy(), res, False, len(log), sweeps, log, exit_rule, p_cur, d_cur)


def solve_deflate(A, k: int, d: int, p: int, X0: np.ndarray, tol: float = 1e-10, maxit: int = 300,
                  s_max: int = 5, w: int | None = None, filter: str = "cheb", arr_method: str = "qr",
                  max_outer: int | None = None, range_digits: float = RANGE_DIGITS) -> SolveResult:
    """Alg. Arrabit2 with continuation (Eq. contin) and deflation (Eq. defl,
    P:1396-1416), MPM sweeps by the dynamic-range rule, fixed p and d (R19):
      tol_1 = sqrt(tol); tol_{t+1} = max(1e-2 tol_t, tol) once max res <= tol_t;
      after every ARR the leading Ritz pairs with res <= max(1e-14, tol_t^2) are locked
      (Q_c, the leading columns of X; at least one pair stays active); the active block
      X is filtered, projected X - Q_c(Q_c^T X) twice and ARR'ed in the
      orthogonal complement of R(Q_c); b = mu_{w_a+1} of the active ARR;
      a final Rayleigh-Ritz on all w columns orders the pairs and recomputes residuals."""
    w = X0.shape[1] if w is None else w
    gamma = None if filter == "cheb" else interp_coeffs(d)
    X = np.array(X0[:, :w], dtype=np.float64, copy=True)
    a = gershgorin_lower(A)
    mu0, _, _ = arr(A, X, 0, method=arr_method)
    b, mu1 = float(mu0[w - 1]), float(mu0[0])
    if not a < b:
        a = b - 1e-8 * (abs(b) + 1.0)
    tol_t = max(tol, math.sqrt(tol))
    nc = 0
    locked_res: list[float] = []
    log = []
    sweeps = 0
    done = False
    limit = maxit if max_outer is None else min(maxit, max_outer)
    for outer in range(1, limit + 1):
        wa = w - nc
        Qc = X[:, :nc]
        Xa = X[:, nc:]
        s = sweeps_rule(mu1, a, b, d, s_max, gamma, range_digits)
        for _ in range(s):
            Xa = mpm_sweep(A, a, b, d, Xa) if gamma is None else poly_sweep(A, a, b, gamma, Xa)
        sweeps += s
        if nc > 0:
            for _ in range(2):
                Xa = Xa - dense.gemm(Qc, dense.gram(Qc, Xa))
        mu, Y, r = arr(A, Xa, p, keep=wa, method=arr_method, Qc=Qc if nc > 0 else None)
        ka = k - nc
        ra = residuals(A, Y[:, :ka], mu[:ka])
        maxres = max(float(np.max(ra)), max(locked_res) if locked_res else 0.0)
        X = np.hstack([Qc, Y[:, :wa]])
        log.append(dict(outer=outer, s=s, a=a, b=b, mu1=float(mu[0]), rank=r, maxres=maxres, locked=nc, tol_t=tol_t))
        if maxres <= tol:
            done = True
            break
        if maxres <= tol_t:
            tol_t = max(1e-2 * tol_t, tol)  # continuation
        b = float(mu[min(wa, r - 1)])
        thr = max(1e-14, tol_t * tol_t)
        add = 0
        while add < ka - 1 and ra[add] <= thr:
            add += 1
        locked_res.extend(float(x) for x in ra[:add])
        nc += add
        mu1 = float(mu[add])
        if not a < b:
            a = b - 1e-8 * (abs(b) + 1.0)
    mu, V = _ritz(A, X)
    Yf = X @ V
    res = residuals(A, Yf[:, :k], mu[:k])
    conv = done and float(np.max(res)) <= tol
    return SolveResult(mu[:k].copy(), Yf[:, :k].copy(), res, conv, len(log), sweeps, log,
                       1 if conv else 0, p, d, nc)
