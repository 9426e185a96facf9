"""ORACLE — test infrastructure only (see oracle/__init__.py).

Plain fp64 CPU implementation of the ARRABIT-MPM hot path, arXiv 1507.06078
(P = /root/reference/PAPER.md line numbers; readings in DESIGN.md §4).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

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
    relative and Alg. poly's Horner output by up to 1e-4 — not a reproducible target."""
    if d < 1:
        raise ValueError("d >= 1")
    t = -np.cos(np.arange(d + 1) * np.pi / d)
    f = np.maximum(0.0, t) ** (10 * d)
    return np.linalg.solve(chebyshev_basis(d, t), f)


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
    Y = X @ np.linalg.inv(X.T @ X)
    Z = cheb_filter(A, a, b, d, Y) if coef is None else poly_filter(A, a, b, coef, Y)
    return Z - X @ (Y.T @ Z - np.eye(X.shape[1])) / 2.0


# --------------------------------------------------------------------------- dense
def orthonormalize(Z: np.ndarray):
    """U in orth(Z) (Alg. RR step 1): equilibrate columns (span unchanged),
    Householder QR with column pivoting (library step), keep
    r = #{i : |R_ii| > n*eps*|R_11|} columns (reading DESIGN.md §4 R8)."""
    Z = np.asarray(Z, dtype=np.float64)
    n, m = Z.shape
    nrm = np.linalg.norm(Z, axis=0)
    keep = nrm > 0
    Zs = Z[:, keep] / nrm[keep]
    if Zs.shape[1] == 0:
        return np.zeros((n, 0)), 0
    Q, R, _ = scipy.linalg.qr(Zs, mode="economic", pivoting=True)
    dR = np.abs(np.diag(R))
    r = int(np.sum(dR > n * np.finfo(float).eps * dR[0]))
    return Q[:, :r], r


def rayleigh_ritz(A, Z: np.ndarray):
    """(Y, Sigma) = RR(A, Z), Alg. RR: U = orth(Z); H = U^T A U;
    H = V^T Sigma V; Y = U V.  Ritz values sorted descending."""
    U, r = orthonormalize(Z)
    AU = spmm(A, U) if r > 0 else np.zeros_like(U)
    H = U.T @ AU
    H = 0.5 * (H + H.T)
    mu, V = np.linalg.eigh(H)
    order = np.argsort(-mu, kind="stable")
    mu = mu[order]
    V = V[:, order]
    return mu, U @ V, r


def arr(A, X: np.ndarray, p: int, keep: int | None = None, rng_seed: int = 12345):
    """(Y, Sigma) = ARR(A, X, p), Alg. ARR: Z = [X, AX, ..., A^p X]
    (plain A, Eq. S:ARR P:515-523), RR(A, Z), keep the leading pairs.
    Returns (mu_all_descending, Y_keep, rank).  If the rank r < keep the block
    is topped up with seeded Gaussian columns orthonormalised against Y
    (reading DESIGN.md §4 R7; never triggered in the pinned cases)."""
    n, w = X.shape
    keep = w if keep is None else keep
    if (p + 1) * w >= n:
        raise ValueError("(p+1)k must be < n (Alg. ARR input, P:536)")
    blocks = [np.asarray(X, dtype=np.float64)]
    for _ in range(p):
        blocks.append(spmm(A, blocks[-1]))
    Z = np.hstack(blocks)
    mu, Y, r = rayleigh_ritz(A, Z)
    if r >= keep:
        return mu, Y[:, :keep], r
    rng = np.random.default_rng(rng_seed)
    extra = rng.standard_normal((n, keep - r))
    extra -= Y @ (Y.T @ extra)
    Q, _ = np.linalg.qr(extra)
    return mu, np.hstack([Y, Q]), r


def residuals(A, Y: np.ndarray, mu: np.ndarray) -> np.ndarray:
    """res_i = ||A y_i - mu_i y_i||_2 / max(1, |mu_i|)  (Eq. resi)."""
    AY = spmm(A, Y)
    R = AY - Y * mu[None, :]
    return col_norms(R) / np.maximum(1.0, np.abs(mu))


def sweeps_rule(mu1: float, a: float, b: float, d: int, s_max: int, gamma=None) -> int:
    """Sweeps between ARR steps (DESIGN.md §4 R6, the dynamic-range rule that
    replaces the paper's rcond inner stop P:1355-1388): amp = |T_d((mu_1-c)/e)|
    (|psi_d((mu_1-c)/e)| with the interpolant filter),
    s = s_max if amp <= 1 else clamp(floor(8/log10(amp)), 1, s_max)."""
    c = 0.5 * (a + b)
    e = 0.5 * (b - a)
    t = (mu1 - c) / e
    amp = abs(float(chebyshev_T(d, t) if gamma is None else psi(gamma, np.array([t]))[0]))
    if not amp > 1.0:
        return s_max
    if not math.isfinite(amp):
        return 1
    return int(min(max(math.floor(8.0 / math.log10(amp)), 1), s_max))


@dataclass
class SolveResult:
    mu: np.ndarray
    Y: np.ndarray
    res: np.ndarray
    converged: bool
    outer: int
    sweeps: int
    log: list = field(default_factory=list)


def solve(A, k: int, d: int, p: int, X0: np.ndarray, tol: float = 1e-10, maxit: int = 300,
          s_max: int = 5, w: int | None = None, max_outer: int | None = None, filter: str = "cheb",
          inner_solver: str = "mpm") -> SolveResult:
    """Fixed-parameter ARRABIT-MPM (Alg. Arrabit2, with the
    adaptive lines disabled; DESIGN.md §4 R3/R6/R10):

        a := Gershgorin lower bound;  U0 := orth(X0); mu := eig(U0^T A U0); b := mu_w
        loop: s := sweeps_rule(mu_1);  s x { X := T_d((A-cI)/e) X; normalise }
              (mu, Y) := ARR(A, X, p)
              res_i, i <= k  (Eq. resi)  ;  stop if max res <= tol              (Eq. out-stop)
              b := mu_{w+1} (monotone once maxres grew);  X := Y[:, :w]   (R3)
    """
    n = A.n
    w = X0.shape[1] if w is None else w  # w - k guard vectors
    gamma = None if filter == "cheb" else interp_coeffs(d)  # "interp": the paper's psi_d (R18)
    X = np.array(X0[:, :w], dtype=np.float64, copy=True)
    a = gershgorin_lower(A)
    mu0, _, _ = rayleigh_ritz(A, X)
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
    for outer in range(1, limit + 1):
        s = sweeps_rule(mu1, a, b, d, s_max, gamma)
        for _ in range(s):
            if inner_solver == "gn":  # Alg. Arrabit2's GN branch
                X = gn_step(A, a, b, d, X, gamma)
            else:
                X = mpm_sweep(A, a, b, d, X) if gamma is None else poly_sweep(A, a, b, gamma, X)
        sweeps += s
        mu, Y, r = arr(A, X, p, keep=w)
        res = residuals(A, Y[:, :k], mu[:k])
        maxres = float(np.max(res))
        log.append(dict(outer=outer, s=s, a=a, b=b, mu1=float(mu[0]), rank=r, maxres=maxres))
        if maxres <= tol:
            return SolveResult(mu[:k].copy(), Y[:, :k].copy(), res, True, outer, sweeps, log)
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
    return SolveResult(mu[:k].copy(), Y[:, :k].copy(), res, False, limit, sweeps, log)
